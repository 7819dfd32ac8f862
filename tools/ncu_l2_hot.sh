# L2 read-hit of the config-5 batched step kernels with and without the evict_last hot prefix.
M=lts__t_sector_op_read_hit_rate.pct,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_hit.sum,lts__t_sectors_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$C > gpurun_out/plain_l2.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:"cheby_batch_(rows|pieces)" -s 2 -c 2 --csv $C > gpurun_out/ncu_l2_hot64.csv 2>gpurun_out/ncu_l2_hot64.err
CPG_HOT_MB=0 ncu --metrics $M --clock-control none -k regex:"cheby_batch_(rows|pieces)" -s 2 -c 2 --csv $C > gpurun_out/ncu_l2_hot0.csv 2>gpurun_out/ncu_l2_hot0.err
grep -h "cheby" gpurun_out/ncu_l2_hot64.csv | cut -d, -f5,13- | head -20
echo ===
grep -h "cheby" gpurun_out/ncu_l2_hot0.csv | cut -d, -f5,13- | head -20
