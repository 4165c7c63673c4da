#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python scripts/pyr_ab.py > gpurun_out/pyr_ab.txt 2>&1
python scripts/pyr_ab.py --dims 256,256,256 --octaves 4 --batch 4 >> gpurun_out/pyr_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "blur or small or brain or large" > gpurun_out/pyr_tests.log 2>&1
tail -2 gpurun_out/pyr_tests.log
if [ "${NCU:-0}" = "1" ]; then
  ncu --set full --import-source on --clock-control none -k regex:blur_xy_plane -c 3 -o gpurun_out/xyplane python scripts/pyr_ab.py --batch 2 > gpurun_out/ncu_xy.log 2>&1
fi
cat gpurun_out/pyr_ab.txt
