#!/bin/bash
# Full measurement session: bench (default args), reference arm, ncu launch
# list of the bench command, DRAM traffic of every pyramid launch of one step.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/full
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/full/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/full/bench_default.jsonl 2> gpurun_out/full/bench_default.err; echo "bench rc=$?"
tail -1 gpurun_out/full/bench_default.jsonl | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/full/bench_reference.jsonl 2> gpurun_out/full/bench_reference.err; echo "ref rc=$?"
tail -1 gpurun_out/full/bench_reference.jsonl | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/full/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/full/launches_run.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/full/pyramid_dram.csv -k regex:"blur3d|detect|orient_kernel|siftrank|order|frame" \
  python scripts/profile_step.py --batch 16 --steps 1 > gpurun_out/full/pyramid_dram.log 2>&1; echo "dram rc=$?"
