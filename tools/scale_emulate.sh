#!/bin/bash
# GPU box: per-rank step times of the C5 strong-scaling sweep on ONE GPU (bench --emulate-shard):
# engine-grouped shards (what bench.py's ranks decide) vs index-contiguous shards (--instances)
cd "$GRAFT_REPO_ROOT" || exit 1
o=gpurun_out/scale_em; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
for N in 2 4 8; do
  for r in 0 $((N-1)); do
    timeout 600 python bench.py --emulate-shard $r/$N --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/em_${r}_${N}.json 2> $o/em_${r}_${N}.err
  done
  timeout 600 python bench.py --instances $((262144 / N)) --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/contig_${N}.json 2> $o/contig_${N}.err
done
for f in $o/em_*.json $o/contig_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['per_kernel_ms']
print('$f'.split('/')[-1], d['config']['instances_per_gpu'], round(d['ms_per_step'],4), 'k1', round(k['k1_project'],3), 'k2', round(k['k2_gbdt'],3), 'k3', round(k['k3_select'],3), 'cells', d['counts_per_step_rank0']['cells'])"; done
