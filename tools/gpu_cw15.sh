#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; }
for cfg in 84 124 123 163 85; do CPG_CW_CFG64=$cfg run c4_g$cfg --config 4 --steps 3 --warmup 3; done
for cfg in 84 124 163; do CPG_CW_CFG64=$cfg run c3_g$cfg --config 3 --mode batched --steps 3 --warmup 3; done
