#!/bin/bash
# Blur iteration: GPU parity tests, stage timing, ncu per-launch pyramid times.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/iter
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/iter/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/iter/pytest_gpu.log
timeout 300 python scripts/stage_bench.py --batch 12 --reps 5 > gpurun_out/iter/stage.log 2>&1; echo "stage rc=$?"
head -1 gpurun_out/iter/stage.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/iter/blur_launches.csv -k regex:"blur|small_oct" python scripts/profile_step.py --batch 12 --steps 1 > gpurun_out/iter/l.log 2>&1; echo "launches rc=$?"
if [ -n "$FULL" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blur3d_stream_kernel" --launch-skip ${SKIP:-5} --launch-count 1 \
  -o gpurun_out/iter/full python scripts/profile_step.py --batch 12 --steps 1 > gpurun_out/iter/f.log 2>&1; echo "full rc=$?"
fi
