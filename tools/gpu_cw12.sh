#!/bin/bash
# Hot prefix x window size with the final geometries (config 5)
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; }
run hw_default --steps 3 --warmup 3
for hot in 48 64 80; do for w in 32 40 48 56; do
  if [ "$hot:$w" != "64:48" ]; then CPG_HOT_MB=$hot CPG_CW_MB=$w run hw_h${hot}_w$w --steps 3 --warmup 3; fi
done; done
CPG_CW_WARM_MB=1280 run hw_warm1280 --steps 3 --warmup 3
CPG_CW_WARM_MB=896 run hw_warm896 --steps 3 --warmup 3
CPG_CW_DEG=4096 run hw_deg4096 --steps 3 --warmup 3
