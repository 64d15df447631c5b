#!/usr/bin/env bash
# A/B: streamed-sweep parity tests, then K1/K2 timing with and without back-projection pieces.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_nonblind_gpu.py tests/test_golden_gpu.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; tail -n 3 gpurun_out/ab_tests.log
for c in 4 2; do
  timeout 600 python scripts/prof_frame.py $c 3 > gpurun_out/ab_prof_$c.log 2>&1; tail -n 1 gpurun_out/ab_prof_$c.log
  PDD_NO_CHAIN=1 timeout 600 python scripts/prof_frame.py $c 3 > gpurun_out/ab_prof_nc_$c.log 2>&1; echo "nochain: $(tail -n 1 gpurun_out/ab_prof_nc_$c.log)"
done
