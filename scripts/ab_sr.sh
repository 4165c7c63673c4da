#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/ab
python scripts/stage_bench.py --batch 16 --reps 3 > gpurun_out/ab/A.log 2>&1; head -1 gpurun_out/ab/A.log
sed -i 's/^__global__ void __launch_bounds__(kSrThreads, 3)$/__global__ void __launch_bounds__(kSrThreads, 2)/' paper_2112_10258_b200/csrc/vk_describe.cu
python -m paper_2112_10258_b200.build --force > gpurun_out/ab/build.log 2>&1
python scripts/stage_bench.py --batch 16 --reps 3 > gpurun_out/ab/B.log 2>&1; head -1 gpurun_out/ab/B.log
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/ab/pytest.log 2>&1; tail -1 gpurun_out/ab/pytest.log
