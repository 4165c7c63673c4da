#!/bin/bash
# A/B of the walk kernels: default build vs variants/libvolkey_<name>.so for each name given (sep_ab: ms + digest).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/walk_ab.txt
: > $out
for i in 1 2; do
  echo "default" >> $out; timeout 300 python scripts/sep_ab.py >> $out 2>&1
  for v in "$@"; do
    echo "$v" >> $out; VK_LIB_PATH=variants/libvolkey_$v.so timeout 300 python scripts/sep_ab.py >> $out 2>&1
  done
done
cat $out
