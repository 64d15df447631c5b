#!/usr/bin/env bash
# One GPU session: parity tests (with the per-config parity report), bench +
# launch list, ncu captures of the two kernels of the iteration (sweep, gather)
# on config 4.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2}
rm -f gpurun_out/parity_$TAG.jsonl
PDD_PARITY_REPORT=gpurun_out/parity_$TAG.jsonl timeout ${TEST_TIMEOUT:-2400} python -m pytest tests/ -q -m gpu > gpurun_out/tests_$TAG.log 2>&1
tail -n 1 gpurun_out/tests_$TAG.log
bash scripts/gpu_bench.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
tail -n 1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_stream -c 1 \
    -o gpurun_out/sweep_$TAG -f python scripts/prof_frame.py 4 1 > gpurun_out/ncu_sweep_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:gather_kernelIf -c 1 \
    -o gpurun_out/gather_$TAG -f python scripts/prof_frame.py 4 1 > gpurun_out/ncu_gather_$TAG.log 2>&1
  tail -n 1 gpurun_out/ncu_sweep_$TAG.log gpurun_out/ncu_gather_$TAG.log
fi
