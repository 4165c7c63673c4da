#!/bin/bash
# A/B: persistent double-buffered (x, y) plane kernel (VK_XY_KERNEL=2) vs the 2-CTA/SM plane kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/xy_stream.txt
: > $out
timeout 300 python scripts/pyr_ab.py --variants 0:0,2:0,0:0,2:0 >> $out 2>&1
for k in 0 2 0 2; do
  echo "VK_XY_KERNEL=$k" >> $out
  VK_XY_KERNEL=$k timeout 300 python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline'].get('frac'), d['e2e']['value'], d.get('rank_parity',{}).get('matches_reference'))" >> $out
done
VK_XY_KERNEL=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_xy_stream.csv timeout 300 python scripts/pyr_ab.py --variants 2:0 --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launch_xy_stream.csv 2>&1 | grep -i blur | head -40 >> $out
cat $out
