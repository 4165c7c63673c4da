#!/bin/bash
# ncu --set full of the R=4 (x, y) plane kernel (octave 0, level 1: no DoG warps) -- issue / stall breakdown.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/prof_xy4
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blur_xy_plane_kernel --launch-skip 1 --launch-count 1 \
  -o $O/xy4 python scripts/profile_step.py --batch 8 --steps 1 > $O/xy.log 2>&1; echo "xy rc=$?"
