# Fused batched kernel: per-launch claim rule (default) vs fixed claims (CPG_CLAIM_ROWS) (GPU box)
for spec in "1 16" "2 16" "2 32" "2 64"; do
  set -- $spec
  for i in 1 2; do
    for cr in rule 4 8; do
      if [ $cr = rule ]; then e=""; else e="CPG_CLAIM_ROWS=$cr"; fi
      env $e python bench.py --no-cpu-baseline --config $1 --mode batched --tile $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$1 tile$2 claim=$cr', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],4))"
    done
  done
done
