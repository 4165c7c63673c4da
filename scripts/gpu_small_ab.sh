#!/bin/bash
# A/B of the small-octaves kernel: pyramid stage time (pyr_ab) for the default build and the given variants,
# then the pyramid parity tests on the default build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
  echo "default"; timeout 300 python scripts/pyr_ab.py --variants 0:0 2>&1 | tail -1
  for v in "$@"; do echo "$v"; VK_LIB_PATH=variants/libvolkey_$v.so timeout 300 python scripts/pyr_ab.py --variants 0:0 2>&1 | tail -1; done
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:small_octaves --csv python scripts/pyr_ab.py --variants 0:0 --reps 1 2>/dev/null | grep small_oct | head -2
for v in "$@"; do VK_LIB_PATH=variants/libvolkey_$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:small_octaves --csv python scripts/pyr_ab.py --variants 0:0 --reps 1 2>/dev/null | grep small_oct | head -1; done
timeout 900 python -m pytest tests -q -m gpu -x -k "brain or pyramid or large or blur or small" 2>&1 | tail -2
