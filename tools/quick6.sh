timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binary.py -m gpu -x -q -k "compact" 2>&1 | tail -2
for wl in C2 C3; do
timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 20 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$wl', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,2), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)})"
done
