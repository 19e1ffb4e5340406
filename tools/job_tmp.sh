cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q -k "compact and (w1 or tiny or parity_configs or shapes)" 2>&1 | tail -2
bash tools/sweep_r02.sh nohint
WL=C5 bash tools/sweep_r02.sh nohint
