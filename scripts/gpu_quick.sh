#!/bin/bash
# Quick GPU iteration: parity tests + per-stage timing.  Logs -> gpurun_out/quick/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/quick/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/quick/pytest_gpu.log
timeout 300 python scripts/stage_bench.py --batch 12 > gpurun_out/quick/stage.log 2>&1; echo "stage rc=$?"
cat gpurun_out/quick/stage.log | tail -4
if [ -n "$BENCH" ]; then timeout 600 python bench.py --no-cpu-baseline > gpurun_out/quick/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/quick/bench.log | cut -c1-600; fi
