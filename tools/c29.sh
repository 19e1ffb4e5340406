cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/t29_all.log 2>&1
tail -3 gpurun_out/t29_all.log
for w in C2 C3; do timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 --steps 50 >> gpurun_out/b29.jsonl; done
timeout 600 python tools/k2_cells_sweep.py C2 20 > gpurun_out/sweep29_C2.txt 2>&1
timeout 600 python tools/k2_cells_sweep.py C3 10 > gpurun_out/sweep29_C3.txt 2>&1
OUT=gpurun_out/prof29_C3; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_project|k3_select_runs" -s 4 -c 2 -o $OUT/full python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/full.log 2>&1
ls -la $OUT
