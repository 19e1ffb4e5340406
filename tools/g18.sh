for wl in C1 C2 C3; do
timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 30 --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$wl', round(d['ms_per_step']*1e3,1), round(d['value']/1e6,2), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)}, 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e6,2))"
done
