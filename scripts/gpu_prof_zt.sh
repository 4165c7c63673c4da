#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/prof_zt
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blur_zt_kernel --launch-skip 5 --launch-count 1 \
  -o $O/zt10 python scripts/profile_step.py --batch 8 --steps 1 > $O/zt.log 2>&1; echo "zt rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blur_xy_plane_kernel --launch-skip 5 --launch-count 1 \
  -o $O/xy10 python scripts/profile_step.py --batch 8 --steps 1 > $O/xy.log 2>&1; echo "xy rc=$?"
