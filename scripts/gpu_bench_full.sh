#!/bin/bash
# Full measurement session: smoke + GPU parity tests, bench (default args),
# reference arm, ncu launch list of the bench command, DRAM traffic of every
# pipeline launch of one 16-volume step, full ncu captures of the hot kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/full
rm -rf $O
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.jsonl 2> $O/bench_default.err; echo "bench rc=$?"
tail -1 $O/bench_default.jsonl | cut -c1-300
if [ -z "$NOREF" ]; then
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.jsonl 2> $O/bench_reference.err; echo "ref rc=$?"
tail -1 $O/bench_reference.jsonl | cut -c1-300
fi
# matching benches before the ncu sessions (a GPU fresh from ncu replays measured 10-30% slow)
timeout 600 python scripts/match_bench.py > $O/match_bench.log 2>&1; echo "match bench rc=$?"
timeout 900 python scripts/database_bench.py 2> $O/database_bench.err | grep "^{" > $O/database_bench.json; echo "database rc=${PIPESTATUS[0]}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-matching > $O/launches_run.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/pyramid_dram.csv -k regex:"blur|small_oct|detect|orient_kernel|siftrank|order|frame" \
  python scripts/profile_step.py --batch 16 --steps 1 > $O/pyramid_dram.log 2>&1; echo "dram rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blur_xy" --launch-skip 5 --launch-count 1 \
  -o $O/blur10_full python scripts/profile_step.py --batch 12 --steps 1 > /dev/null 2>&1; echo "blur full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"match_i8_ws" -o $O/match_full \
  python scripts/match_prof.py > /dev/null 2>&1; echo "match full rc=$?"
for k in siftrank_kernel orient_kernel; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-count 1 \
  -o $O/${k}_full python scripts/profile_step.py --batch 12 --steps 1 > /dev/null 2>&1; echo "$k full rc=$?"
done
