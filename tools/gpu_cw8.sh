#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; }
run s_default --steps 3 --warmup 3
CPG_CW_SPREAD=4 run s_block --steps 3 --warmup 3
CPG_CW_SPREAD=4 CPG_CW_MB=40 run s_block_40mb --steps 3 --warmup 3
CPG_CW_SPREAD=4 CPG_CW_MB=32 run s_block_32mb --steps 3 --warmup 3
CPG_CW_SPREAD=4 CPG_CW_CFG=841 run s_block_84 --steps 3 --warmup 3
