#!/bin/bash
# compute-sanitizer on the round-2 kernels: warp-specialised matcher (TMA + mbarrier ring), keypoint ordering
# (chunk sort), refinement, fused orientation + SIFT-Rank.  Logs -> gpurun_out/san/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/san
mkdir -p $O
for tool in ${MATCH_TOOLS:-memcheck racecheck synccheck}; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=match_i8_ws --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "nn_tensor_core" > $O/match_$tool.log 2>&1; echo "match $tool rc=$?"; tail -2 $O/match_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 \
  python -m pytest tests/test_gpu_refine.py -q -x > $O/detect_memcheck.log 2>&1; echo "detect memcheck rc=$?"; tail -2 $O/detect_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --kernel-name kns=chunk_sort_kernel --print-limit 20 \
  python -m pytest tests/test_gpu_refine.py -q -x > $O/sort_racecheck.log 2>&1; echo "sort racecheck rc=$?"; tail -2 $O/sort_racecheck.log
timeout 1500 compute-sanitizer --tool memcheck --kernel-name kns=orsr --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "fused_orientation and 2.5" > $O/orsr_memcheck.log 2>&1; echo "orsr memcheck rc=$?"; tail -2 $O/orsr_memcheck.log
