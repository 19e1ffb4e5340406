#!/bin/bash
# round-2 quick check on the GPU box: compact-path parity, scale parity, smoke, C5 bench
cd "$GRAFT_REPO_ROOT" || exit 1
o=gpurun_out/r02/${1:-q1}; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "compact or scale or multirank" > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $o/bench_c5.json 2> $o/bench_c5.err
timeout 600 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_c3.json 2> $o/bench_c3.err
timeout 600 python bench.py --workload C2 --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_c2.json 2> $o/bench_c2.err
tail -3 $o/pytest.log; tail -2 $o/smoke.log; cut -c1-400 $o/bench_c5.json; tail -3 $o/bench_c5.err
