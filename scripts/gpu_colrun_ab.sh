#!/bin/bash
# A/B: running y-pass offsets (VK_COL_RUNNING=1, default build) vs per-access address arithmetic (variant).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/colrun_ab.txt
: > $out
for i in 1 2; do
  echo "new" >> $out; timeout 300 python scripts/pyr_ab.py --variants 0:0 >> $out 2>&1
  echo "old" >> $out; VK_LIB_PATH=variants/libvolkey_colrun0.so timeout 300 python scripts/pyr_ab.py --variants 0:0 >> $out 2>&1
done
for i in 1 2; do
  echo "bench new" >> $out; timeout 300 python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline'].get('frac'), d['e2e']['value'], d.get('rank_parity',{}).get('matches_reference'))" >> $out
  echo "bench old" >> $out; VK_LIB_PATH=variants/libvolkey_colrun0.so timeout 300 python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline'].get('frac'), d['e2e']['value'], d.get('rank_parity',{}).get('matches_reference'))" >> $out
done
cat $out
