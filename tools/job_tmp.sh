cd "$GRAFT_REPO_ROOT"
o=gpurun_out/r02/q13; mkdir -p $o
timeout 1500 python bench.py --workload C4 > $o/bench_c4.json 2> $o/bench_c4.err; tail -3 $o/bench_c4.err; python -c "
import json; d=json.load(open('$o/bench_c4.json'))
for k in ['value','steps','ms_per_step','drained','blocked_requests_at_end','arrival_phase','round_ms_pctl','replay_stats']: print(k, d.get(k))
print(d['config']['timed']); print(d['e2e'])"
