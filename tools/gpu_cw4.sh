#!/bin/bash
mkdir -p gpurun_out/cw
python -m pytest tests/test_gpu_column_windows.py -x -q 2>&1 | tail -5
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "import json; d=json.load(open('gpurun_out/cw/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/cw/$name.log; }
run base3 --steps 3 --warmup 3
export CPG_CW_DEG=2048 CPG_CW_MB=48 CPG_CW_WARM_MB=1024
run rp83 --steps 3 --warmup 3
CPG_CW_CFG=830 run norp83 --steps 3 --warmup 3
CPG_CW_CFG=841 run rp84 --steps 3 --warmup 3
CPG_CW_CFG=1631 run rp163 --steps 3 --warmup 3
CPG_CW_DEG=1024 CPG_CW_MB=32 run rp83_deg1024_32 --steps 3 --warmup 3
CPG_CW_WARM_MB=2048 run rp83_warm2g --steps 3 --warmup 3
CPG_CW_MB=40 run rp83_40mb --steps 3 --warmup 3
