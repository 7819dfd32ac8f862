#!/bin/bash
mkdir -p gpurun_out/cw
python -m pytest tests/test_gpu_column_windows.py -x -q 2>&1 | tail -15 > gpurun_out/cw/tests.txt
cat gpurun_out/cw/tests.txt
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "import json; d=json.load(open('gpurun_out/cw/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/cw/$name.log; grep "column-window" gpurun_out/cw/$name.log | head -2; }
export CPG_CW_DEBUG=1
run base --steps 3 --warmup 3
CPG_CW_DEG=4096 run cw4096 --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_SPREAD=0 run cw4096_nospread --steps 3 --warmup 3
CPG_CW_DEG=8192 run cw8192 --steps 3 --warmup 3
CPG_CW_DEG=2048 run cw2048 --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_MB=48 run cw4096_48mb --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_MB=16 run cw4096_16mb --steps 3 --warmup 3
CPG_CW_DEG=4096 CPG_CW_WARM_MB=1024 run cw4096_warm1g --steps 3 --warmup 3
