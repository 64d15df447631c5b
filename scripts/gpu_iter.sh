#!/usr/bin/env bash
# Quick GPU iteration: parity tests + per-kernel profile of c1/c4 (+ optional ncu)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_nonblind_gpu.py -q -m gpu -x > gpurun_out/t_gpu.log 2>&1
tail -n 3 gpurun_out/t_gpu.log
for c in 1 4; do timeout 600 python scripts/prof_frame.py $c 3 > gpurun_out/prof_plain_$c.log 2>&1; tail -n 1 gpurun_out/prof_plain_$c.log; done
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_stream -c 1 \
    -o gpurun_out/prof_c4 -f python scripts/prof_frame.py 4 1 > gpurun_out/ncu_c4.log 2>&1
  tail -n 2 gpurun_out/ncu_c4.log
fi
