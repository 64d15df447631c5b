#!/usr/bin/env bash
# Bench (default config 4), then the ncu launch list of the same command.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1
tail -n 1 gpurun_out/bench_$TAG.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_small_$TAG.log 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch_$TAG.log 2>&1
tail -n 2 gpurun_out/ncu_launch_$TAG.log
