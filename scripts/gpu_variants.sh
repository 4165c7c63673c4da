#!/bin/bash
# pyr_ab on the default library and each variants/libvolkey_*.so (VARIANTS="a b c")
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/variants.txt
echo "default" > $out
python scripts/pyr_ab.py --variants ${PV:-0:0} >> $out 2>&1
for v in $VARIANTS; do
  echo "variant $v" >> $out
  VK_LIB_PATH=variants/libvolkey_$v.so python scripts/pyr_ab.py --variants ${PV:-0:0} >> $out 2>&1
done
cat $out
