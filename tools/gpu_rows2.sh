#!/bin/bash
mkdir -p gpurun_out/rows
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/rows/$name.json 2> gpurun_out/rows/$name.log; python -c "
import json; d=json.load(open('gpurun_out/rows/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/rows/$name.log; }
run p_default --steps 3 --warmup 3
for cfg in 841 1041 1031 1231 1631; do CPG_CW_CFG=$cfg run p_cw$cfg --steps 3 --warmup 3; done
