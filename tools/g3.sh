timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_binary.py -m gpu -x -q -k "cells or fused or compact or decide or ctx" 2>&1 | tail -15 > gpurun_out/g4_pytest.log
timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/g4_c2.json 2> gpurun_out/g4_c2.err
timeout 600 python bench.py --workload C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g4_c3.json 2> gpurun_out/g4_c3.err
cat gpurun_out/g4_pytest.log; tail -n 3 gpurun_out/g4_c2.err gpurun_out/g4_c3.err
python - <<'PY'
import json
for f in ["gpurun_out/g4_c2.json","gpurun_out/g4_c3.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["per_kernel_ms"], d["roofline"]["frac"], d["e2e"]["value"], d["e2e"]["matches_device_path"])
    except Exception as e: print(f, e)
PY
bash tools/profile_compact.sh C3 r01e > /dev/null 2>&1
bash tools/profile_compact.sh C2 r01e > /dev/null 2>&1
ls gpurun_out/prof_r01e_C3 gpurun_out/prof_r01e_C2
