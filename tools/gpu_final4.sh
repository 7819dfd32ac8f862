#!/bin/bash
# Bounds-checked build over every kernel path and the GPU suite on the final build; three repeats of the default bench.
bash tools/checked.sh gpurun_out/checked > gpurun_out/checked_summary.txt 2>&1
cat gpurun_out/checked_summary.txt | cut -c1-160
unset CPG_LIB_PATH
mkdir -p gpurun_out/repeat
for i in 1 2 3; do python bench.py --no-cpu-baseline > gpurun_out/repeat/default_$i.json 2> gpurun_out/repeat/default_$i.log; python -c "
import json; d=json.load(open('gpurun_out/repeat/default_$i.json')); print('default run $i', round(d['value'],1), round(d['e2e']['value'],1), d['steps'], d['warmup'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
python bench.py --impl reference > gpurun_out/repeat/reference.json 2> gpurun_out/repeat/reference.log; tail -c 600 gpurun_out/repeat/reference.json
