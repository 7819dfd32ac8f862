#!/bin/bash
mkdir -p gpurun_out/cw
python -m pytest tests/test_gpu_column_windows.py -x -q 2>&1 | tail -5
run() { name=$1; shift; python bench.py --no-cpu-baseline "$@" > gpurun_out/cw/$name.json 2> gpurun_out/cw/$name.log; python -c "import json; d=json.load(open('gpurun_out/cw/$name.json')); print('$name', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],3))" || tail -3 gpurun_out/cw/$name.log; }
run base4 --steps 3 --warmup 3
export CPG_CW_DEG=2048 CPG_CW_MB=48 CPG_CW_WARM_MB=1024
CPG_CW_CFG=830 run w_plain83 --steps 3 --warmup 3
run w_plain_rp83 --steps 3 --warmup 3
CPG_CW_CFG=84 run w_plain84 --steps 3 --warmup 3
CPG_CW_CFG=830 CPG_CW_MB=32 run w_plain83_32mb --steps 3 --warmup 3
CPG_CW_CFG=830 CPG_CW_DEG=1024 CPG_CW_MB=32 run w_plain83_deg1024_32mb --steps 3 --warmup 3
CPG_CW_CFG=830 CPG_CW_WARM_MB=2048 run w_plain83_warm2g --steps 3 --warmup 3
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
M="dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.avg.per_cycle_active"
CPG_CW_CFG=830 ncu --metrics $M --clock-control none -k regex:"cheby_batch_pieces" -s 3 -c 1 $C 2>&1 | grep -E "cheby_batch|dram__|gpu__time|hit_rate|inst_executed|warps_active|long_scoreboard|throughput"
