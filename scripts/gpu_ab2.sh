#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
V=paper_2011_00162_b200/variants
timeout 900 python -m pytest tests/test_nonblind_gpu.py tests/test_blind_gpu.py tests/test_golden_gpu.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; tail -n 2 gpurun_out/ab_tests.log
for c in 4 2 3 1; do
  echo "cur c$c: $(timeout 600 python scripts/prof_frame.py $c 3 2>&1 | tail -n 1)"
  echo "cur-nochain c$c: $(PDD_NO_CHAIN=1 timeout 600 python scripts/prof_frame.py $c 3 2>&1 | tail -n 1)"
done
for n in 1 2 3; do
  echo "stage64 c3: $(PDD_LIB=$V/stage64.so timeout 300 python scripts/prof_frame.py 3 3 2>&1 | tail -n 1)"
  echo "stage64 notma c3: $(PDD_NO_TMA_ROWS=1 PDD_LIB=$V/stage64.so timeout 300 python scripts/prof_frame.py 3 3 2>&1 | tail -n 1)"
done
