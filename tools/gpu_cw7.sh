#!/bin/bash
mkdir -p gpurun_out/cw
python -m pytest tests/test_gpu_column_windows.py -x -q 2>&1 | tail -3
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; grep "column-window" gpurun_out/cw/$name.log | head -1; }
export CPG_CW_DEBUG=1
run h_default --steps 3 --warmup 3
CPG_CW_HUB=512 run h512_cut2048 --steps 3 --warmup 3
CPG_CW_HUB=512 CPG_CW_DEG=512 run h512_cut512 --steps 3 --warmup 3
CPG_CW_HUB=128 CPG_CW_DEG=512 run h128_cut512 --steps 3 --warmup 3
CPG_CW_HUB=128 CPG_CW_DEG=128 run h128_cut128 --steps 3 --warmup 3
CPG_CW_HUB=512 CPG_CW_DEG=512 CPG_CW_SPREAD=2 run h512_cut512_sorted --steps 3 --warmup 3
