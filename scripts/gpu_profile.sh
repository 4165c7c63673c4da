#!/bin/bash
# ncu launch list + full captures of the top kernels.  Logs -> gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
B=${B:-8}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python scripts/profile_step.py --batch $B --steps 1 > gpurun_out/launches_run.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:blur3d_ring_kernel -s 5 -c 1 \
  -o gpurun_out/blur_r10 python scripts/profile_step.py --batch $B --steps 1 > gpurun_out/prof_blur.log 2>&1
echo "blur rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"orient_kernel|siftrank_kernel|detect_kernel" -c 3 \
  -o gpurun_out/desc python scripts/profile_step.py --batch $B --steps 1 > gpurun_out/prof_desc.log 2>&1
echo "desc rc=$?"
ls -la gpurun_out
