#!/bin/bash
mkdir -p gpurun_out/sharded
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/sharded/$name.json 2> gpurun_out/sharded/$name.log; python -c "
import json; d=json.load(open('gpurun_out/sharded/$name.json'))
print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline'].get('step',d['roofline'])['launch_ms'],3), d['config']['parallelism'], d['config']['allgather'], d['config']['sparse_early_steps'])" || tail -5 gpurun_out/sharded/$name.log; }
run plain --steps 3 --warmup 3
run sharded_c1 --sharded --steps 3 --warmup 3
CPG_CHUNKS=4 run sharded_c4 --sharded --steps 3 --warmup 3
CPG_CHUNKS=4 CPG_CW_DEG=0 run sharded_c4_nocw --sharded --steps 3 --warmup 3
CPG_CW_DEG=0 run sharded_c1_nocw --sharded --steps 3 --warmup 3
