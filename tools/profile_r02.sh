#!/bin/bash
# GPU box: launch list + ncu --set full of the compact path's kernels at one workload
# usage: tools/profile_r02.sh WORKLOAD TAG [extra bench args]
cd "$GRAFT_REPO_ROOT" || exit 1
WL=${1:-C3}; TAG=${2:-r02a}
OUT=gpurun_out/prof_${TAG}_${WL}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${@:3}"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches.log 2>&1
ncu --set full --clock-control none -k regex:"k1_packed|k1_compact|k1_cells_collect|k3_compact|k2_cells_phase" -s 6 -c 6 -o $OUT/full $B > $OUT/full.log 2>&1
ls -la $OUT
