#!/usr/bin/env bash
# A/B of variants on the S = 64 shapes (configs 1, 3): parity tests, then
# nonblind iteration timing and the blind bench line per variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
V=${V:-"base s64 nofuse"}
for v in $V; do
  so=paper_2011_00162_b200/variants/$v.so
  r=$(PDD_LIB=$so timeout 600 python -m pytest tests/test_nonblind_gpu.py tests/test_blind_gpu.py -q -m gpu -k "streamed or pieces or one_sweep or blind" 2>&1 | tail -n 1)
  echo "$v tests: $r"
done
for rep in 1 2; do
  for v in $V; do
    so=paper_2011_00162_b200/variants/$v.so
    echo "$v c3: $(PDD_LIB=$so timeout 600 python scripts/prof_frame.py 3 20 2>&1 | tail -n 1)"
    echo "$v c1: $(PDD_LIB=$so timeout 600 python scripts/prof_frame.py 1 20 2>&1 | tail -n 1)"
    echo "$v c4: $(PDD_LIB=$so timeout 600 python scripts/prof_frame.py 4 5 2>&1 | tail -n 1)"
  done
done
for v in $V; do
  so=paper_2011_00162_b200/variants/$v.so
  echo "$v c3 blind: $(PDD_LIB=$so timeout 600 python bench.py --config 3 --no-e2e --no-cpu-baseline 2>&1 | tail -n 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done
