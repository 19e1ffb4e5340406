#!/bin/bash
# GPU box: bench per libtp variant (TP_LIB_PATH) or env setting ("env:VAR=VAL"), kernel times
# usage: WL=C3 tools/sweep_r02.sh [variant|env:VAR=VAL] ...
cd "$GRAFT_REPO_ROOT" || exit 1
WL=${WL:-C3}
for v in base "$@"; do
  case $v in
    base) L="";;
    env:*) L="${v#env:}";;
    *) L="TP_LIB_PATH=paper_2408_05235_b200/libtp_$v.so";;
  esac
  env $L timeout 600 python bench.py --workload $WL --no-cpu-baseline --steps 10 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $WL', round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['per_kernel_ms'].items() if not isinstance(v,str)})"
done
