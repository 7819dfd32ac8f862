# A/B of the batched step's fused vs split kernels (CPG_BATCH_SPLIT) per config (run on the GPU box)
for spec in "2 64" "3 64" "4 64"; do
  set -- $spec
  for i in 1 2; do
    for sp in default 0 1; do
      if [ $sp = default ]; then e=""; else e="CPG_BATCH_SPLIT=$sp"; fi
      env $e python bench.py --no-cpu-baseline --config $1 --mode batched --tile $2 --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$1 tile$2 split=$sp', round(d['value'],1), round(d['roofline']['launch_ms'],4))"
    done
  done
done
