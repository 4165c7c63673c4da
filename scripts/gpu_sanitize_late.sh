#!/bin/bash
# compute-sanitizer on the late round-2 changes: the plane blur (running y-pass offsets), the persistent
# two-group plane kernel, the orientation walk (pair_ok bitset, by-value fallback).  Logs -> gpurun_out/san2/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/san2
mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "xy_kernels or blur_fused or blur_all" > $O/blur_memcheck.log 2>&1; echo "blur memcheck rc=$?"; tail -2 $O/blur_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --kernel-name kns=blur_xy --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "xy_kernels" > $O/xy_racecheck.log 2>&1; echo "xy racecheck rc=$?"; tail -2 $O/xy_racecheck.log
timeout 1500 compute-sanitizer --tool memcheck --kernel-name kns=orient_kernel --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -k "brain" > $O/orient_memcheck.log 2>&1; echo "orient memcheck rc=$?"; tail -2 $O/orient_memcheck.log
