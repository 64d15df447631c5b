#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for L in default 1 2 3 4 6 8; do
  if [ $L = default ]; then e=""; else e="PDD_PIECE_LEN=$L"; fi
  echo "c4 L=$L: $(env $e timeout 600 python scripts/prof_frame.py 4 3 2>&1 | tail -n 1)"
done
for L in default 2 4; do
  if [ $L = default ]; then e=""; else e="PDD_PIECE_LEN=$L"; fi
  echo "c2 L=$L: $(env $e timeout 600 python scripts/prof_frame.py 2 3 2>&1 | tail -n 1)"
done
