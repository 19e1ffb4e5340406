for kb in 200 100 220; do
  TP_K2_PHASE_KB=$kb timeout 300 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('phaseKB $kb', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
done
for w in 2 4 8; do
  TP_K3C_WARPS=$w timeout 300 python bench.py --no-cpu-baseline --steps 50 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('k3w $w', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
done
