#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
V=paper_2011_00162_b200/variants
for n in 1 2 3; do
  echo "stage64pad c3: $(PDD_LIB=$V/stage64pad.so timeout 300 python scripts/prof_frame.py 3 3 2>&1 | tail -n 1)"
  echo "stage64pad c1: $(PDD_LIB=$V/stage64pad.so timeout 300 python scripts/prof_frame.py 1 3 2>&1 | tail -n 1)"
done
for n in 1 2 3 4; do
  echo "cur streamed tests: $(timeout 300 python -m pytest tests/test_nonblind_gpu.py tests/test_blind_gpu.py -q -m gpu -k 'streamed' 2>&1 | tail -n 1)"
done
