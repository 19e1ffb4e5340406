cd "$GRAFT_REPO_ROOT"
o=gpurun_out/r02/q6; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -x -q -k "compact or scale or binary or admission or replay" > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
tail -3 $o/pytest.log
bash tools/sweep_r02.sh m4 m6
WL=C5 bash tools/sweep_r02.sh
WL=C2 bash tools/sweep_r02.sh
