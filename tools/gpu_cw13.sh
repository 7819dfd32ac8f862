#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; }
run hx_default --steps 3 --warmup 3
for hot in 32 40 48; do for w in 56 64 72; do CPG_HOT_MB=$hot CPG_CW_MB=$w run hx_h${hot}_w$w --steps 3 --warmup 3; done; done
run hx_default2 --steps 3 --warmup 3
CPG_HOT_MB=48 CPG_CW_MB=56 run c4_h48_w56 --config 4 --steps 3 --warmup 3
run c4_default --config 4 --steps 3 --warmup 3
CPG_HOT_MB=48 CPG_CW_MB=56 run c3_h48_w56 --config 3 --mode batched --steps 3 --warmup 3
run c3_default --config 3 --mode batched --steps 3 --warmup 3
