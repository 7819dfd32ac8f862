# ncu --set full of the sparse early-step kernels (scan + fill) of config 5, B = 16, M = 2
mkdir -p gpurun_out/ncu_masked
CMD="python tools/step_times.py --config 5 --mode batched --M 2 --reps 1"
$CMD > gpurun_out/ncu_masked/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cheby_sparse" -c 4 \
    -o gpurun_out/ncu_masked/c5_sparse $CMD > gpurun_out/ncu_masked/ncu.log 2>&1
