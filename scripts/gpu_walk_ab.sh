#!/bin/bash
# A/B of the walk kernels: default build vs variants/libvolkey_${1:-head}.so (sep_ab: ms + output digest).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/walk_ab.txt
: > $out
for i in 1 2 3; do
  echo "new" >> $out; timeout 300 python scripts/sep_ab.py >> $out 2>&1
  echo "${1:-head}" >> $out; VK_LIB_PATH=variants/libvolkey_${1:-head}.so timeout 300 python scripts/sep_ab.py >> $out 2>&1
done
cat $out
