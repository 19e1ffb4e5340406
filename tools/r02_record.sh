#!/bin/bash
# GPU box: record run (tools/r02_final.sh) + C5 launch list and ncu --set full summary / traffic json
# (the report itself is deleted on the box: gpurun copies back at most 64 MiB)
# usage: tools/r02_record.sh TAG
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${1:-rec}
bash tools/r02_final.sh $TAG
bash tools/profile_r02.sh C5 $TAG
P=gpurun_out/prof_${TAG}_C5
python tools/ncu_summary.py $P/full.ncu-rep > $P/ncu_summary.txt 2>&1
python tools/traffic_json.py $P/full.ncu-rep C5 > $P/traffic.log 2>&1
cp profiles/traffic_C5.json $P/traffic_C5.json
rm -f $P/full.ncu-rep
ls -la $P
