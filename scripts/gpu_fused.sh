#!/bin/bash
# Fused orientation + SIFT-Rank: A/B + parity + GPU tests.  Logs -> gpurun_out/fused/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/fused
mkdir -p $O
timeout 300 python scripts/fused_ab.py --batch 8 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -4 $O/ab.log
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
fi
if [ -n "$BENCH" ]; then
timeout 600 python bench.py --no-cpu-baseline --no-extras --no-matching > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?"
tail -1 $O/bench.jsonl | cut -c1-400
fi
