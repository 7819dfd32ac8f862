# fused (CPG_BATCH_SPLIT=0) vs split (1) batched kernels on configs 1-3 with the round-2 build.
for cfg in "1" "2" "3 --mode batched --tile 64"; do
  for rep in 1 2; do
    for sp in 0 1; do
      CPG_BATCH_SPLIT=$sp python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg split=$sp', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1))"
    done
  done
done
