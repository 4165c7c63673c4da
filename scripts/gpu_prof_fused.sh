#!/bin/bash
# ncu of the fused orientation + SIFT-Rank kernel (and the separate pair for comparison), 8 volumes.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/prof_fused
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"orsr_kernel" -c 1 -o $O/orsr \
  python scripts/profile_step.py --batch 8 --steps 1 > $O/orsr.log 2>&1; echo "orsr rc=$?"
if [ -z "$NOSEP" ]; then
VK_FUSED=0 timeout 900 ncu --set full --clock-control none -k regex:"orient_kernel|siftrank_kernel" -c 2 -o $O/sep \
  python scripts/profile_step.py --batch 8 --steps 1 > $O/sep.log 2>&1; echo "sep rc=$?"
fi
