#!/bin/bash
# GPU box: K2 rows per lane (TP_K2_RU_CELLS) at C2, an N = 8 engine shard, C3 and C5
cd "$GRAFT_REPO_ROOT" || exit 1
for v in 2 1; do
  for a in "--workload C2" "--emulate-shard 0/8" "--workload C3" "--workload C5"; do
    TP_K2_RU_CELLS=$v timeout 600 python bench.py $a --no-cpu-baseline --steps 10 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('RU=$v', '$a', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)}, 'k2frac', round(d['roofline']['per_kernel']['k2']['frac'],3))"
  done
done
