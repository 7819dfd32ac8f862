#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "import json; d=json.load(open('gpurun_out/cw/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/cw/$name.log; }
export CPG_CW_DEG=2048 CPG_CW_MB=48 CPG_CW_WARM_MB=1024
run g83 --steps 3 --warmup 3
CPG_CW_SPREAD=2 run g83_sorted --steps 3 --warmup 3
for cfg in 84 85 162 163 44 46; do CPG_CW_CFG=$cfg run g$cfg --steps 3 --warmup 3; done
CPG_CW_CFG=84 CPG_CW_SPREAD=2 run g84_sorted --steps 3 --warmup 3
CPG_CW_CFG=162 CPG_CW_SPREAD=2 run g162_sorted --steps 3 --warmup 3
CPG_CW_WARM_MB=2048 run g83_warm2g --steps 3 --warmup 3
CPG_CW_DEG=1024 run g83_deg1024 --steps 3 --warmup 3
