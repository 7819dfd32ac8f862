#!/bin/bash
mkdir -p gpurun_out/small
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/small/$name.json 2> gpurun_out/small/$name.log; python -c "
import json; d=json.load(open('gpurun_out/small/$name.json'))
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],4))" || tail -3 gpurun_out/small/$name.log; }
for i in 1 2; do
run c1_default --config 1 --steps 8 --warmup 4
CPG_HOT_MB=0 run c1_hot0 --config 1 --steps 8 --warmup 4
run c2_default --config 2 --steps 8 --warmup 4
CPG_HOT_MB=0 run c2_hot0 --config 2 --steps 8 --warmup 4
done
