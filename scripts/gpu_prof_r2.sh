#!/bin/bash
# ncu captures of the round-2 hot kernels: orient_kernel, siftrank_kernel (8 volumes), the warp-specialised matcher.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/prof_r2
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"orient_kernel|siftrank_kernel" -c 2 -o $O/walks \
  python scripts/profile_step.py --batch 8 --steps 1 > $O/walks.log 2>&1; echo "walks rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"match_i8_ws" -c 1 -o $O/match_ws \
  python scripts/match_prof.py > $O/match.log 2>&1; echo "match rc=$?"
