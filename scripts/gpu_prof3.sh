#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"blur3d_ring_kernel" -s 5 -c 1 -o gpurun_out/blur3 python scripts/profile_step.py --batch 16 --steps 1 > gpurun_out/prof_blur.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"orient_kernel|siftrank_kernel" -c 2 -o gpurun_out/desc6 python scripts/profile_step.py --batch 8 --steps 1 > gpurun_out/prof_desc.log 2>&1
python scripts/stage_bench.py --batch 16 --reps 3 > gpurun_out/stage.log 2>&1; cat gpurun_out/stage.log
