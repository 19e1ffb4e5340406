for v in m4p4 m5p4 m6p4 m3p8; do
  TP_LIB_PATH=paper_2408_05235_b200/libtp_$v.so timeout 300 python bench.py --workload C3 --no-cpu-baseline --steps 5 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
done
TP_LIB_PATH=paper_2408_05235_b200/libtp_m4p4.so timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 m4p4', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
