#!/bin/bash
# Run ON THE GPU BOX (via gpurun): launch list + ncu full captures of the default bench step.
# Usage: tools/profile_gpu.sh [workload] [tag] [k2 variant]
set -u
WL=${1:-C2}
TAG=${2:-r01}
K2=${3:-fused}
OUT=gpurun_out/prof_${TAG}_${WL}_${K2}
mkdir -p $OUT
BENCH="python bench.py --workload $WL --k2 $K2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
# 1) every launch with its device time (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/launches.log 2>&1
# 2) full set on every kernel of one step (skip the warm-up launches)
ncu --set full --clock-control none --import-source on -k regex:"k1_project|k2_runs|k2_gbdt|k2_expand|k3_select" -s 12 -c 5 -o $OUT/full $BENCH > $OUT/full.log 2>&1
ls -la $OUT
