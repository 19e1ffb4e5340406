#!/bin/bash
# GPU box: launch list + ncu full on k1_project / k2_runs / k3_select_runs at C3
OUT=gpurun_out/prof_${1:-r01}_C3
mkdir -p $OUT
B="python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > $OUT/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_project|k2_runs|k3_select_runs|k2_gbdt" -s 5 -c 4 -o $OUT/full $B > $OUT/full.log 2>&1
ls -la $OUT
