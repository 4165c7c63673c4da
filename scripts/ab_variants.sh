#!/bin/bash
# A/B of compile-time variants: VARIANTS="name:sed-expression;..." applied to vk_describe.cu / vk_orient.cu
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ab2
cp paper_2112_10258_b200/csrc/vk_describe.cu /tmp/desc.orig
cp paper_2112_10258_b200/csrc/vk_orient.cu /tmp/orient.orig
python scripts/stage_bench.py --batch 12 --reps 3 2>&1 | grep "exact_only=False" | sed 's/^/base: /'
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name="${v%%:*}"; expr="${v#*:}"
  cp /tmp/desc.orig paper_2112_10258_b200/csrc/vk_describe.cu; cp /tmp/orient.orig paper_2112_10258_b200/csrc/vk_orient.cu
  sed -i "$expr" paper_2112_10258_b200/csrc/vk_describe.cu paper_2112_10258_b200/csrc/vk_orient.cu
  python -m paper_2112_10258_b200.build --force > gpurun_out/ab2/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
  python scripts/stage_bench.py --batch 12 --reps 3 2>&1 | grep "exact_only=False" | sed "s/^/$name: /"
done
