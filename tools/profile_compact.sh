#!/bin/bash
# GPU box: ncu full on the compact path's kernels (k1_compact, k2_gbdt, k3_compact) at one workload
WL=${1:-C3}; TAG=${2:-r01c}
OUT=gpurun_out/prof_${TAG}_${WL}
mkdir -p $OUT
B="python bench.py --workload $WL --k2 compact --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_packed|k1_compact|k3_compact|k2_cells_phase" -s 5 -c 5 -o $OUT/full $B > $OUT/full.log 2>&1
ls -la $OUT
