#!/bin/bash
# GPU box: C3 / C5 bench per libtp variant (TP_LIB_PATH), kernel times
cd "$GRAFT_REPO_ROOT" || exit 1
WL=${WL:-C3}
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L="TP_LIB_PATH=paper_2408_05235_b200/libtp_$v.so"; fi
  env $L timeout 600 python bench.py --workload $WL --no-cpu-baseline --steps 10 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $WL', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)})"
done
