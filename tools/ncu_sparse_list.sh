# ncu launch list (time, DRAM bytes, instructions) of the sparse early-step kernels of config 5, B = 16, M = 2
mkdir -p gpurun_out/ncu_sparse
CMD="python tools/step_times.py --config 5 --mode batched --M 2 --reps 1"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"cheby_sparse|coarsen|first_push|init_onehot" -c 12 --csv \
    --log-file gpurun_out/ncu_sparse/c5_M2_list.csv $CMD > gpurun_out/ncu_sparse/ncu.log 2>&1
cat gpurun_out/ncu_sparse/c5_M2_list.csv | cut -d, -f5,12- | tail -40
