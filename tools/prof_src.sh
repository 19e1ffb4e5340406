#!/bin/bash
# GPU box: ncu --set full (with source) of the named kernels at one workload, for per-line SASS counts
# usage: tools/prof_src.sh WORKLOAD TAG REGEX [extra bench args]
cd "$GRAFT_REPO_ROOT" || exit 1
WL=${1:-C3}; TAG=${2:-src}; RX=${3:-"k1_packed|k3_compact"}
OUT=gpurun_out/prof_${TAG}_${WL}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --workload $WL --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph ${@:4}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 3 -c 2 -o $OUT/full $B > $OUT/full.log 2>&1
ls -la $OUT; tail -3 $OUT/full.log
