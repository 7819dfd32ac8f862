#!/bin/bash
mkdir -p gpurun_out/cw
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; }
run hy_default --steps 3 --warmup 3
export CPG_ROWS_HOT_MB=64
for hot in 8 16 24 32; do for w in 48 56; do CPG_HOT_MB=$hot CPG_CW_MB=$w run hy_h${hot}_w${w}_rows64 --steps 3 --warmup 3; done; done
CPG_HOT_MB=32 CPG_CW_MB=56 CPG_ROWS_HOT_MB=80 run hy_h32_w56_rows80 --steps 3 --warmup 3
CPG_HOT_MB=32 CPG_CW_MB=56 CPG_ROWS_HOT_MB=96 run hy_h32_w56_rows96 --steps 3 --warmup 3
CPG_HOT_MB=32 CPG_CW_MB=56 run c4_h32_w56_rows64 --config 4 --steps 3 --warmup 3
CPG_HOT_MB=16 CPG_CW_MB=56 run c4_h16_w56_rows64 --config 4 --steps 3 --warmup 3
CPG_HOT_MB=32 CPG_CW_MB=56 run c3_h32_w56_rows64 --config 3 --mode batched --steps 3 --warmup 3
