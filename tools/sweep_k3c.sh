for v in base m6 m7; do
  if [ $v = base ]; then L=""; else L="TP_LIB_PATH=paper_2408_05235_b200/libtp_$v.so"; fi
  env $L timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 10 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v C3', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)})"
done
