for k1 in 1 2; do for k3 in 1 2 4; do
TP_K1C_WARPS=$k1 TP_K3C_WARPS=$k3 timeout 600 python bench.py --workload C4 --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4 k1 $k1 k3 $k3', round(d['value']/1e6,3), d['per_round_ms'])"
done; done
for k1 in 1 2; do for k3 in 1 2; do
TP_K1C_WARPS=$k1 TP_K3C_WARPS=$k3 timeout 600 python bench.py --workload C3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3 k1 $k1 k3 $k3', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
done; done
