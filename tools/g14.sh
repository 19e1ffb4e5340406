timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binary.py tests/test_gpu_replay.py -m gpu -x -q -k "compact or decide or ctx or replay" 2>&1 | tail -3
for wpi in 1 2 4; do
TP_K1C_WARPS=$wpi timeout 300 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 wpi $wpi', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
done
timeout 300 python bench.py --workload C3 --no-cpu-baseline --steps 5 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
