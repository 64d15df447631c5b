#!/usr/bin/env bash
# A/B of kernel variants (paper_2011_00162_b200/variants/*.so): streamed-sweep
# parity tests, then config-4 (and config-2) iteration timing per variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
V=${V:-"base tw half twhalf"}
for v in $V; do
  so=paper_2011_00162_b200/variants/$v.so
  r=$(PDD_LIB=$so timeout 600 python -m pytest tests/test_nonblind_gpu.py -q -m gpu -k "streamed or pieces or one_sweep" 2>&1 | tail -n 1)
  echo "$v tests: $r"
done
for rep in 1 2; do
  for v in $V; do
    so=paper_2011_00162_b200/variants/$v.so
    echo "$v c4: $(PDD_LIB=$so timeout 600 python scripts/prof_frame.py 4 5 2>&1 | tail -n 1)"
  done
done
for v in $V; do
  so=paper_2011_00162_b200/variants/$v.so
  echo "$v c2: $(PDD_LIB=$so timeout 600 python scripts/prof_frame.py 2 5 2>&1 | tail -n 1)"
done
