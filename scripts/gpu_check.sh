#!/bin/bash
# One GPU session: exhaustive sqrt sweep, the GPU test suite, one default bench line.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/sqrt_approx_err.cu -o /tmp/sq && timeout 120 /tmp/sq > gpurun_out/sqrt_sweep.txt 2>&1
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if [ "${RUN_BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
fi
tail -3 gpurun_out/pytest_gpu.log
tail -c 3000 gpurun_out/bench.jsonl
