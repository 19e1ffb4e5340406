# multi-rank bench path on one GPU (gloo collectives; TP_BENCH_DIST_TEST=1 test aid)
for wl in C2 C5; do
TP_BENCH_DIST_TEST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --workload $wl --steps 5 --warmup 3 --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl x2', d['n_gpus'], round(d['value']/1e6,2), d['config']['global_instances'], d['config']['parallelism'], d['e2e']['matches_device_path'], d['scaling'])"
done
