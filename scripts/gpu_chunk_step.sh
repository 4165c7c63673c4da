cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/chunk_step.txt
: > $out
for ch in 0 1 2 4 0; do
  echo "chunk=$ch" >> $out
  VK_PYR_CHUNK=$ch python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline'].get('frac'), d['e2e']['value'])" >> $out
done
cat $out
