#!/bin/bash
# Round-1 record run (one B200): GPU tests, smoke, default bench (C2), C3/C4/C5 bench lines,
# launch list + ncu full capture of the default bench step.
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/final/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_c2.json 2> gpurun_out/final/bench_c2.err
timeout 900 python bench.py --workload C3 --steps 10 --warmup 3 > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
timeout 900 python bench.py --workload C4 --steps 20 --warmup 3 > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/final/bench_c5.json 2> gpurun_out/final/bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c2.csv $B > gpurun_out/final/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_compact|k3_compact|k2_cells_phase" -s 4 -c 4 -o gpurun_out/final/full_c2 $B > gpurun_out/final/full.log 2>&1
cat gpurun_out/final/pytest.log gpurun_out/final/smoke.log
for f in gpurun_out/final/bench_*.json; do echo $f; tail -c 600 $f; echo; done
