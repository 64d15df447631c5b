#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
A=tests/test_dropin_gpu.py::test_reference_pybind_frontend_routes_to_the_gpu_library
B="tests/test_nonblind_gpu.py::test_streamed_sweep_large_frames_matches_oracle"
timeout 900 python -m pytest $A "$B" -x -q -m gpu > gpurun_out/dbg3_ab.log 2>&1; tail -n 2 gpurun_out/dbg3_ab.log
CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest $A "$B" -x -q -m gpu > gpurun_out/dbg3_ab_blk.log 2>&1; tail -n 2 gpurun_out/dbg3_ab_blk.log
grep -m3 -B30 "CudaError:" gpurun_out/dbg3_ab_blk.log | head -80
timeout 900 compute-sanitizer --print-limit 10 python -m pytest $A "$B" -x -q -m gpu > gpurun_out/dbg3_san.log 2>&1; grep -m 30 -E "=====" gpurun_out/dbg3_san.log | head -40
