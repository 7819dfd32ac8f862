#!/bin/bash
mkdir -p gpurun_out/cw
python -m pytest tests/test_gpu_column_windows.py tests/test_gpu_sharded_loopback.py -x -q 2>&1 | tail -5
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "
import json; d=json.load(open('gpurun_out/cw/$name.json')); k=d['roofline'].get('kernels',{})
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), [round(v['launch_ms'],2) for v in k.values()])" || tail -3 gpurun_out/cw/$name.log; }
run rh_default --steps 3 --warmup 3
for mb in 32 48 80 96 112; do CPG_ROWS_HOT_MB=$mb run rh_$mb --steps 3 --warmup 3; done
CPG_ROWS_RP=1 CPG_ROWS_HOT_MB=96 run rh_96_rp --steps 3 --warmup 3
python bench.py --sharded --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/cw/sharded1.json 2> gpurun_out/cw/sharded1.log; python -c "
import json; d=json.load(open('gpurun_out/cw/sharded1.json')); print('sharded(1 rank)', round(d['value'],1), round(d['e2e']['value'],1), d['config']['parallelism'], d['config']['allgather'])" || tail -5 gpurun_out/cw/sharded1.log
