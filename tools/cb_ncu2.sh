M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
for deg in 0 4096; do
CPG_CB_DEG=$deg ncu --metrics $M --clock-control none -k regex:cheby_batch_pieces -s 3 -c 1 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/cb2_ncu_$deg.txt 2>&1
echo "== CB_DEG=$deg"; grep -E "^ +[a-z_]+__" gpurun_out/cb2_ncu_$deg.txt
done
