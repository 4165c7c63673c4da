#!/bin/bash
# Per-stage timings (stage_bench) on the default library and variants/libvolkey_$v.so; parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/stage_ab.txt
echo "default" > $out
python scripts/stage_bench.py --batch 8 --reps 3 >> $out 2>&1
for v in $VARIANTS; do
  echo "variant $v" >> $out
  VK_LIB_PATH=variants/libvolkey_$v.so python scripts/stage_bench.py --batch 8 --reps 3 >> $out 2>&1
done
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_known_answers.py -q -x > gpurun_out/stage_tests.log 2>&1
  tail -3 gpurun_out/stage_tests.log >> $out
fi
if [ -n "${NCU_K:-}" ]; then
  ncu --set full --import-source on --clock-control none -k regex:$NCU_K -s ${NCU_S:-2} -c 1 -o gpurun_out/stage_full python scripts/stage_bench.py --batch 8 --reps 1 > gpurun_out/ncu_stage.log 2>&1
fi
cat $out
