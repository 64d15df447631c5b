#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_nonblind_gpu.py -x -q -m gpu > gpurun_out/dbg2_nb.log 2>&1; tail -n 3 gpurun_out/dbg2_nb.log
timeout 900 python -m pytest tests/test_nccl_gpu.py tests/test_nonblind_gpu.py -x -q -m gpu -k "nccl or one_sweep or streamed" > gpurun_out/dbg2_nccl_nb.log 2>&1; tail -n 3 gpurun_out/dbg2_nccl_nb.log
CUDA_LAUNCH_BLOCKING=1 timeout 1200 python -m pytest tests/test_blind_gpu.py tests/test_golden_gpu.py tests/test_lagrangian_gpu.py tests/test_nccl_gpu.py tests/test_nonblind_gpu.py -x -q -m gpu > gpurun_out/dbg2_blocking.log 2>&1; tail -n 3 gpurun_out/dbg2_blocking.log
grep -m3 -B5 "CudaError:" gpurun_out/dbg2_blocking.log
