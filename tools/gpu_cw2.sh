#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "import json; d=json.load(open('gpurun_out/cw/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/cw/$name.log; grep "column-window" gpurun_out/cw/$name.log | head -1; }
export CPG_CW_DEBUG=1 CPG_CW_SPREAD=0
run base2 --steps 3 --warmup 3
CPG_CW_DEG=4096 run s0_4096 --steps 3 --warmup 3
CPG_CW_DEG=2048 run s0_2048 --steps 3 --warmup 3
CPG_CW_DEG=8192 run s0_8192 --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_MB=48 run s0_4096_48mb --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_MB=24 run s0_4096_24mb --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_MB=16 run s0_4096_16mb --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_WARM_MB=1024 run s0_4096_warm1g --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_WARM_MB=256 run s0_4096_warm256 --steps 3 --warmup 3
CPG_CW_DEG=2048 CPG_CW_MB=48 run s0_2048_48mb --steps 3 --warmup 3
CPG_CW_DEG=2048 CPG_CW_MB=48 CPG_CW_WARM_MB=1024 run s0_2048_48mb_warm1g --steps 3 --warmup 3
