#!/bin/bash
# GPU box, one optimisation iteration: build, compact-path parity subset, C5/C3 bench lines,
# ncu --set full (with source) of the named kernels at C5.
# usage: tools/iter.sh TAG [REGEX] [PYTEST_K]
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${1:-it}; RX=${2:-"k1_packed|k3_compact"}; PK=${3:-"compact or scale"}
o=gpurun_out/it/$TAG; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "$PK" > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_c5.json 2> $o/bench_c5.err
timeout 600 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_c3.json 2> $o/bench_c3.err
if [ "$RX" != "none" ]; then
B="python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 3 -c 2 -o $o/full $B > $o/ncu.log 2>&1
fi
tail -2 $o/pytest.log; python tools/bsum.py $o/bench_c5.json $o/bench_c3.json
