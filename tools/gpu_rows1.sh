#!/bin/bash
mkdir -p gpurun_out/rows
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/rows/$name.json 2> gpurun_out/rows/$name.log; python -c "
import json; d=json.load(open('gpurun_out/rows/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/rows/$name.log; }
run r_default --steps 3 --warmup 3
export CPG_ROWS_RP=1
for cfg in 83 84 104 123 163; do CPG_ROWS_RP_CFG=$cfg run r_rp$cfg --steps 3 --warmup 3; done
