#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2112_10258_b200.build
python scripts/pyr_ab.py > gpurun_out/pyr_ab.txt 2>&1
python scripts/pyr_ab.py --dims 256,256,256 --octaves 4 --batch 4 >> gpurun_out/pyr_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "blur or small or brain or large" > gpurun_out/pyr_tests.log 2>&1
tail -2 gpurun_out/pyr_tests.log
for v in 0 1; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_v$v.csv python scripts/pyr_ab.py --variants $v --reps 1 > /dev/null 2>&1
done
python scripts/launch_table.py gpurun_out/launch_v0.csv > gpurun_out/launch_v0.txt 2>&1
python scripts/launch_table.py gpurun_out/launch_v1.csv > gpurun_out/launch_v1.txt 2>&1
if [ "${NCU:-0}" = "1" ]; then
  ncu --set full --import-source on --clock-control none -k regex:blur_xy_plane -s 6 -c 2 -o gpurun_out/xyplane python scripts/pyr_ab.py --variants 0 --reps 1 > gpurun_out/ncu_xy.log 2>&1
fi
cat gpurun_out/pyr_ab.txt
head -30 gpurun_out/launch_v0.txt
