#!/usr/bin/env bash
# All GPU tests, each file bounded by its own timeout.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for t in tests/test_*_gpu.py; do
  n=$(basename $t .py)
  timeout 900 python -m pytest $t -q -m gpu > gpurun_out/$n.log 2>&1
  echo "$n: $(tail -n 1 gpurun_out/$n.log)"
done
