#!/bin/bash
# Full-step bench A/B over env settings: CONFIGS="name:ENV=1,ENV2=0;name2:..."
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/bench_ab.txt
: > $out
IFS=';' read -ra CS <<< "$CONFIGS"
for c in "${CS[@]}"; do
  name="${c%%:*}"; envs="${c#*:}"
  env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-matching --no-extras ${BENCH_ARGS:-} > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  python - "$name" gpurun_out/bench_$name.json >> $out <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["stages_ms_per_step"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
cat $out
