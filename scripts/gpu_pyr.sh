#!/bin/bash
# Pyramid A/B (xy:z kernel variants), parity tests of the blur, launch table of the default variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2112_10258_b200.build
python scripts/pyr_ab.py ${PYR_ARGS:-} > gpurun_out/pyr_ab.txt 2>&1
python scripts/pyr_ab.py --dims 256,256,256 --octaves 4 --batch 4 ${PYR_ARGS:-} >> gpurun_out/pyr_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x > gpurun_out/pyr_tests.log 2>&1
tail -2 gpurun_out/pyr_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_v0.csv python scripts/pyr_ab.py --variants 0:0 --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launch_v0.csv > gpurun_out/launch_v0.txt 2>&1
if [ "${NCU:-0}" = "1" ]; then
  ncu --set full --import-source on --clock-control none -k regex:${NCU_K:-blur_z4} -s ${NCU_S:-5} -c 1 -o gpurun_out/pyr_full python scripts/pyr_ab.py --variants 0:0 --reps 1 > gpurun_out/ncu_pyr.log 2>&1
fi
cat gpurun_out/pyr_ab.txt
grep -A20 "by kernel" gpurun_out/launch_v0.txt
