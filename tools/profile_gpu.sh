#!/bin/bash
# Run ON THE GPU BOX (via gpurun): launch list + ncu full captures of the three kernels.
# Usage: tools/profile_gpu.sh [workload] [tag]
set -u
WL=${1:-C2}
TAG=${2:-r01}
OUT=gpurun_out/prof_${TAG}_${WL}
mkdir -p $OUT
BENCH="python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
# 1) every launch with its device time (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/launches.log 2>&1
# 2) full set on the dominant kernel (K2) and on K1/K3
ncu --set full --clock-control none --import-source on -k regex:k2_gbdt -s 3 -c 1 -o $OUT/k2_full $BENCH > $OUT/k2_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_project|k3_select" -s 6 -c 2 -o $OUT/k13_full $BENCH > $OUT/k13_full.log 2>&1
ls -la $OUT
