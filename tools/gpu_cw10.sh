#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; grep "column-window" gpurun_out/cw/$name.log | head -1; }
export CPG_CW_DEBUG=1
run c4_default --config 4 --steps 3 --warmup 3
CPG_CW_HUB=1024 run c4_hub1024 --config 4 --steps 3 --warmup 3
CPG_CW_HUB=1024 CPG_CW_DEG=1024 run c4_hub1024_cut1024 --config 4 --steps 3 --warmup 3
CPG_CW_HUB=512 CPG_CW_DEG=512 run c4_hub512_cut512 --config 4 --steps 3 --warmup 3
CPG_CW_HUB=256 CPG_CW_DEG=256 run c4_hub256_cut256 --config 4 --steps 3 --warmup 3
CPG_CW_MB=32 run c4_32mb --config 4 --steps 3 --warmup 3
CPG_CW_WARM_MB=2048 run c4_warm2g --config 4 --steps 3 --warmup 3
run c3_default --config 3 --mode batched --steps 3 --warmup 3
CPG_CW_HUB=256 CPG_CW_DEG=256 run c3_hub256_cut256 --config 3 --mode batched --steps 3 --warmup 3
CPG_CW_HUB=512 CPG_CW_DEG=512 CPG_CW_WARM_MB=2560 run c3_hub512_cut512_warmall --config 3 --mode batched --steps 3 --warmup 3
