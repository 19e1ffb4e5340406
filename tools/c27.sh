cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_binary.py -x -q --timeout 300 > gpurun_out/t27_binary.log 2>&1
tail -3 gpurun_out/t27_binary.log
for w in C2 C3; do for s in exhaustive binary; do
 timeout 300 python bench.py --workload $w --search $s --no-cpu-baseline >> gpurun_out/b27.jsonl 2>gpurun_out/b27_$w_$s.err
done; done
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/t27_all.log 2>&1
tail -3 gpurun_out/t27_all.log
