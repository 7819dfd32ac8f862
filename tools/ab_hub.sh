# A/B of the fused batched kernel's hub piece length (CPG_FUSED_HUB_EDGES) on the
# small-graph configs: tools/ab_hub.sh <lib.so>...   (run on the GPU box)
mkdir -p gpurun_out
for cfg in 1 2; do
 for i in 1 2; do
  for lib in paper_2412_10789_b200/libcpg.so "$@"; do
    CPG_LIB_PATH=$lib python bench.py --no-cpu-baseline --config $cfg --mode batched 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$cfg', '$lib', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],4))"
  done
 done
done
