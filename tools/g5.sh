timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/g5_pytest.log
timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/g5_c2.json 2> gpurun_out/g5_c2.err
timeout 600 python bench.py --workload C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g5_c3.json 2> gpurun_out/g5_c3.err
timeout 600 python bench.py --workload C4 --steps 20 --warmup 3 > gpurun_out/g5_c4.json 2> gpurun_out/g5_c4.err
cat gpurun_out/g5_pytest.log; tail -n 3 gpurun_out/g5_c2.err gpurun_out/g5_c3.err gpurun_out/g5_c4.err
python - <<'PY'
import json
for f in ["gpurun_out/g5_c2.json","gpurun_out/g5_c3.json","gpurun_out/g5_c4.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d.get("per_kernel_ms", d.get("per_round_ms")), d.get("roofline",{}).get("frac"), (d.get("e2e") or {}).get("value"))
    except Exception as e: print(f, e)
PY
