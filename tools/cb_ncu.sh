M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum
CPG_CB_DEBUG=1 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>&1 | tail -3
for deg in 0 32768; do
CPG_CB_DEG=$deg ncu --metrics $M --clock-control none -k regex:cheby_batch -s 6 -c 4 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/cb_ncu_$deg.txt 2>&1
grep -E "cheby_batch|gpu__time|dram__bytes|hit_rate|srcunit" gpurun_out/cb_ncu_$deg.txt
done
