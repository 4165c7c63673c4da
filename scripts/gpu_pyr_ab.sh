#!/bin/bash
# Pyramid stage A/B: default build vs variants/libvolkey_<name>.so (pyr_ab, 2 rounds).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
  echo "default"; timeout 300 python scripts/pyr_ab.py --variants 0:0 2>&1 | tail -1
  for v in "$@"; do echo "$v"; VK_LIB_PATH=variants/libvolkey_$v.so timeout 300 python scripts/pyr_ab.py --variants 0:0 2>&1 | tail -1; done
done
