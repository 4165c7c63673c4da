#!/bin/bash
# Pyramid volume-chunk x z-chunk sweep (L2 residency of the intermediate), one process per setting.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/chunk_sweep.txt
: > $out
for ch in 8 4 2 1; do
  for mc in 6 3; do
    echo "chunk=$ch zmin=$mc" >> $out
    VK_PYR_CHUNK=$ch VK_ZT_MINCHUNK=$mc python scripts/pyr_ab.py --variants 0:0 >> $out 2>&1
  done
done
VK_PYR_CHUNK=${NCU_CHUNK:-2} VK_Z_MINCHUNK=${NCU_ZMIN:-4} ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/launch_chunk.csv python scripts/pyr_ab.py --variants 0:0 --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launch_chunk.csv > gpurun_out/launch_chunk.txt 2>&1
cat $out
tail -12 gpurun_out/launch_chunk.txt
