for v in m6p2 m8p2 m6p4 m8p4; do
  TP_LIB_PATH=paper_2408_05235_b200/libtp_$v.so timeout 300 python bench.py --workload C3 --no-cpu-baseline --steps 5 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
done
timeout 300 python bench.py --workload C3 --no-cpu-baseline --steps 5 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base(k1 fast)', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items()})"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_admission.py tests/test_gpu_replay.py -m gpu -x -q -k "compact or decide or replay or admission" 2>&1 | tail -3
