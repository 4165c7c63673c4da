#!/bin/bash
# Step A/B (bench value, no side measurements): default build vs variants/libvolkey_<name>.so, alternating.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then lib=""; else lib="variants/libvolkey_$v.so"; fi
    VK_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-matching --no-cpu-baseline --no-e2e 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['value'], d['stages_ms_per_step'], d['rank_parity']['matches_reference'])"
  done
done
