#!/bin/bash
# Round-2 check session: exhaustive sqrt.approx sweep, GPU tests, a short bench.  Logs -> gpurun_out/check2/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/check2
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/sqrt_approx_err.cu -o /tmp/sq && timeout 300 /tmp/sq > $O/sqrt_approx_sweep.txt 2>&1; echo "sqrt rc=$?"; cat $O/sqrt_approx_sweep.txt
timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-matching > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?"
tail -1 $O/bench.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['stages_ms_per_step'], d.get('configs3',{}).get('volumes_per_s'), d.get('dropin',{}).get('ms_per_call'))"
