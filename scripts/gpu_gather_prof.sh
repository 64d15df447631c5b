#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python scripts/prof_frame.py 4 2 > gpurun_out/pp.log 2>&1 &&
timeout 900 ncu --set full --clock-control none -k regex:gather_kernel -c 1 \
  -o gpurun_out/prof_gather_c4 -f python scripts/prof_frame.py 4 1 > gpurun_out/ncu_gather.log 2>&1
tail -n 2 gpurun_out/ncu_gather.log
