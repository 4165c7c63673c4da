#!/bin/bash
# ncu: per-launch times of every pyramid launch of one 12-volume step, and a
# full-set capture of the radius-10 and radius-5 blur launches of octave 0.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/prof/blur_launches.csv -k regex:"blur3d|small_oct" python scripts/profile_step.py --batch 12 --steps 1 > gpurun_out/prof/l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blur3d_stream_kernel" --launch-skip 5 --launch-count 1 \
  -o gpurun_out/prof/blur10 python scripts/profile_step.py --batch 12 --steps 1 > gpurun_out/prof/f.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blur3d_stream_kernel" --launch-skip 2 --launch-count 1 \
  -o gpurun_out/prof/blur5 python scripts/profile_step.py --batch 12 --steps 1 > gpurun_out/prof/f5.log 2>&1; echo "full5 rc=$?"
