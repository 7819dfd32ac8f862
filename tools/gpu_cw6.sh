#!/bin/bash
mkdir -p gpurun_out/cw
python -m pytest tests/test_gpu_column_windows.py -x -q 2>&1 | tail -3
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "import json; d=json.load(open('gpurun_out/cw/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/cw/$name.log; }
CPG_ROWS_RP=1 run base_rowsrp --steps 3 --warmup 3
export CPG_CW_DEG=2048 CPG_CW_MB=48 CPG_CW_WARM_MB=1024
run cw_rp --steps 3 --warmup 3
CPG_ROWS_RP=1 run cw_rp_rowsrp --steps 3 --warmup 3
CPG_ROWS_RP=1 CPG_CW_CFG=841 run cw_rp84_rowsrp --steps 3 --warmup 3
CPG_ROWS_RP=1 CPG_CW_MB=32 run cw_rp_rowsrp_32mb --steps 3 --warmup 3
CPG_ROWS_RP=1 CPG_CW_MB=40 run cw_rp_rowsrp_40mb --steps 3 --warmup 3
CPG_ROWS_RP=1 CPG_CW_DEG=1024 run cw_rp_rowsrp_deg1024 --steps 3 --warmup 3
CPG_ROWS_RP=1 CPG_CW_WARM_MB=1536 run cw_rp_rowsrp_warm1536 --steps 3 --warmup 3
CPG_ROWS_RP=1 CPG_CW_WARM_MB=768 run cw_rp_rowsrp_warm768 --steps 3 --warmup 3
unset CPG_CW_DEG
run c4_base --config 4 --steps 3 --warmup 3
CPG_ROWS_RP=1 run c4_rowsrp --config 4 --steps 3 --warmup 3
CPG_CW_DEG=2048 CPG_ROWS_RP=1 run c4_cw --config 4 --steps 3 --warmup 3
run c3_base --config 3 --mode batched --steps 3 --warmup 3
CPG_CW_DEG=2048 CPG_ROWS_RP=1 run c3_cw --config 3 --mode batched --steps 3 --warmup 3
