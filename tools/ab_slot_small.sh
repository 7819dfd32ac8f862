# Fused batched kernel geometry (CPG_SLOT_CFG = U*10 + CTAs/SM) on the small-graph configs (GPU box)
for cfg in 1 2; do
  for i in 1 2; do
    for sc in 0 41 45 46 64 85; do
      CPG_SLOT_CFG=$sc python bench.py --no-cpu-baseline --config $cfg --mode batched 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$cfg slot=$sc', round(d['value'],1), round(d['roofline']['launch_ms'],4))"
    done
  done
done
