#!/bin/bash
# GPU box: full gpu suite + smoke + default bench (the driver's round-end sequence) + C2/C3 lines
cd "$GRAFT_REPO_ROOT" || exit 1
o=gpurun_out/r02/${1:-full}; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 600 python bench.py > $o/bench_default.json 2> $o/bench_default.err
timeout 600 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_c3.json 2> $o/bench_c3.err
timeout 600 python bench.py --workload C2 --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_c2.json 2> $o/bench_c2.err
tail -3 $o/pytest.log; tail -2 $o/smoke.log; cut -c1-300 $o/bench_default.json; tail -3 $o/bench_default.err
