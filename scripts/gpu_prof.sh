#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${1:-4}
timeout 600 python scripts/prof_frame.py $CFG 2 > gpurun_out/prof_plain_$CFG.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -c 1 \
  -o gpurun_out/prof_c$CFG -f python scripts/prof_frame.py $CFG 1 > gpurun_out/ncu_c$CFG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c$CFG.csv python scripts/prof_frame.py $CFG 2 > /dev/null 2>&1
tail -3 gpurun_out/prof_plain_$CFG.log gpurun_out/ncu_c$CFG.log
