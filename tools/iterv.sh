#!/bin/bash
# GPU box: parity subset, C5/C3 sweep over libtp variants, ncu (with source) of the base build at C5
# usage: tools/iterv.sh TAG REGEX "PYTEST_K" variant...
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=$1; RX=$2; PK=$3; shift 3
o=gpurun_out/it/$TAG; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q -k "$PK" > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/pytest.log
tail -2 $o/pytest.log
WL=C5 bash tools/sweep_r02.sh "$@" 2>&1 | tee $o/sweep_c5.txt
WL=C3 bash tools/sweep_r02.sh "$@" 2>&1 | tee $o/sweep_c3.txt
WL=C2 bash tools/sweep_r02.sh "$@" 2>&1 | tee $o/sweep_c2.txt
if [ "$RX" != "none" ]; then
B="python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 3 -c 1 -o $o/full $B > $o/ncu.log 2>&1
fi
