#!/usr/bin/env bash
# Debug session: one failing test under compute-sanitizer, quick parity, K1/K2 timing on c4.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${T:-"tests/test_nonblind_gpu.py::test_streamed_sweep_large_frames_matches_oracle"}
timeout 600 python -m pytest "$T" -x -q -m gpu > gpurun_out/dbg_plain.log 2>&1; tail -n 3 gpurun_out/dbg_plain.log
timeout 900 compute-sanitizer --print-limit 20 python -m pytest "$T" -x -q -m gpu > gpurun_out/dbg_san.log 2>&1; grep -m 20 -E "Invalid|Error|error|at 0x|by thread|kernel" gpurun_out/dbg_san.log | head -30
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -m gpu > gpurun_out/dbg_ops.log 2>&1; tail -n 3 gpurun_out/dbg_ops.log
for c in 4 2; do timeout 600 python scripts/prof_frame.py $c 3 > gpurun_out/dbg_prof_$c.log 2>&1; tail -n 1 gpurun_out/dbg_prof_$c.log; done
