cd "$GRAFT_REPO_ROOT"
o=gpurun_out/r02/q8; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
tail -3 $o/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 900 python bench.py > $o/bench_c5.json 2> $o/bench_c5.err; cut -c1-300 $o/bench_c5.json
timeout 600 python bench.py --workload C3 --no-cpu-baseline > $o/bench_c3.json 2> $o/bench_c3.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline > $o/bench_c2.json 2> $o/bench_c2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $o/bench_ref.json 2> $o/bench_ref.err; cut -c1-200 $o/bench_ref.json
