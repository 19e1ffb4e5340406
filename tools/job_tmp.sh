cd "$GRAFT_REPO_ROOT"
o=gpurun_out/r02/q10; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q -k "replay" > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
tail -2 $o/pytest.log
timeout 1200 python bench.py --workload C4 > $o/bench_c4.json 2> $o/bench_c4.err; tail -5 $o/bench_c4.err; cut -c1-1500 $o/bench_c4.json
