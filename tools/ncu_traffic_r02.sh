# ncu --set full captures of the step kernels of configs 2, 3 (batched and single) and 4 (after a
# plain run of the same command line): DRAM bytes per step for bench.py's roofline basis.
set -x
C2="python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline"
$C2 > gpurun_out/plain_c2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:cheby_batch_kernel -s 20 -c 1 -o gpurun_out/prof_c2 $C2 > gpurun_out/ncu_c2.log 2>&1
C3="python bench.py --config 3 --mode batched --tile 64 --steps 1 --warmup 1 --no-cpu-baseline"
$C3 > gpurun_out/plain_c3b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"cheby_batch_(pieces|rows)" -s 4 -c 2 -o gpurun_out/prof_c3b $C3 > gpurun_out/ncu_c3b.log 2>&1
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline"
$C4 > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"cheby_batch_(pieces|rows)" -s 4 -c 2 -o gpurun_out/prof_c4 $C4 > gpurun_out/ncu_c4.log 2>&1
C3S="python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline"
$C3S > gpurun_out/plain_c3s.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:cheby_step_kernel -s 30 -c 1 -o gpurun_out/prof_c3s $C3S > gpurun_out/ncu_c3s.log 2>&1
ls -la gpurun_out/*.ncu-rep
