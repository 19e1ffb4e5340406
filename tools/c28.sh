cd $GRAFT_REPO_ROOT
for v in ut2 default ut8; do for w in C2 C3; do
  if [ $v = default ]; then L=""; else L="TP_LIB_PATH=paper_2408_05235_b200/libtp_$v.so"; fi
  env $L timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 --steps 50 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/b28.jsonl
done; done
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/t28_all.log 2>&1
tail -3 gpurun_out/t28_all.log
