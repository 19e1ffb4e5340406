#!/bin/bash
# GPU box: full gpu suite + smoke + default bench + C3/C2/C4 lines + reference arm
cd "$GRAFT_REPO_ROOT" || exit 1
o=gpurun_out/r02/${1:-final}; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 600 python bench.py > $o/bench_c5.json 2> $o/bench_c5.err
timeout 600 python bench.py --workload C3 > $o/bench_c3.json 2> $o/bench_c3.err
timeout 600 python bench.py --workload C2 > $o/bench_c2.json 2> $o/bench_c2.err
timeout 900 python bench.py --workload C4 > $o/bench_c4.json 2> $o/bench_c4.err
timeout 600 python bench.py --impl reference > $o/bench_ref.json 2> $o/bench_ref.err
tail -3 $o/pytest.log; tail -2 $o/smoke.log; python tools/bsum.py $o/bench_c5.json $o/bench_c3.json $o/bench_c2.json; cut -c1-300 $o/bench_c4.json; cut -c1-300 $o/bench_ref.json
