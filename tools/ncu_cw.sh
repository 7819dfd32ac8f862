#!/bin/bash
# ncu of the piece kernel: uniform pieces vs column-window pieces
mkdir -p gpurun_out/cw_ncu
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
export CPG_CW_SPREAD=0
ncu --metrics $M --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 $C > gpurun_out/cw_ncu/base.txt 2>&1
CPG_CW_DEG=4096 CPG_CW_WARM_MB=1024 ncu --metrics $M --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 $C > gpurun_out/cw_ncu/cw4096_warm1g.txt 2>&1
CPG_CW_DEG=2048 CPG_CW_MB=48 CPG_CW_WARM_MB=1024 ncu --metrics $M --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 $C > gpurun_out/cw_ncu/cw2048_48_warm1g.txt 2>&1
grep -E "cheby_batch|dram__bytes_read|gpu__time|hit_rate|inst_executed|warps_active|long_scoreboard|lts__throughput" gpurun_out/cw_ncu/*.txt
