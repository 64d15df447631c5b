#!/usr/bin/env bash
# GPU-box check: parity tests, then benches (each bounded by its own timeout).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_ops_gpu.py -q -m gpu > gpurun_out/t_ops.log 2>&1
timeout 1500 python -m pytest tests/test_nonblind_gpu.py -q -m gpu > gpurun_out/t_nb.log 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1
timeout 1200 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/b4.log 2>&1
for f in gpurun_out/t_ops.log gpurun_out/t_nb.log gpurun_out/b1.log gpurun_out/b4.log; do echo "== $f"; tail -n 4 "$f"; done
