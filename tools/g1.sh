set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/g1_bench_c2.json 2> gpurun_out/g1_bench_c2.err
timeout 900 python bench.py --workload C3 --steps 5 --warmup 3 > gpurun_out/g1_bench_c3.json 2> gpurun_out/g1_bench_c3.err
timeout 900 python bench.py --workload C4 --steps 20 --warmup 3 > gpurun_out/g1_bench_c4.json 2> gpurun_out/g1_bench_c4.err
cat gpurun_out/g1_pytest.log gpurun_out/g1_smoke.log gpurun_out/g1_bench_c2.json gpurun_out/g1_bench_c3.json gpurun_out/g1_bench_c4.json
