timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binary.py tests/test_gpu_admission.py tests/test_gpu_replay.py -m gpu -x -q -k "compact or decide or ctx or admission or replay or c1_sweep or full_size" 2>&1 | tail -3
for wl in C2 C3; do
timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 30 --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$wl', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,2), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)}, 'frac', round(d['roofline']['frac'],3))"
done
TP_K1C_PACKED=0 timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 10 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3 unpacked', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)})"
