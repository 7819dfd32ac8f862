# Final round-2 build: ncu launch list of the default bench, then ncu --set full captures of the
# split batched step kernels of configs 5, 4 and 3 (each after a plain run of the same command).
mkdir -p gpurun_out/final
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$C > gpurun_out/final/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c5.csv $C > gpurun_out/final/ncu_list.log 2>&1
echo "launch list rc=$?"
# full captures skip the two sparse early steps of the first tile (-s: the 4th and 5th piece/row launches are full steps)
$C > gpurun_out/final/plain_c5b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 -o gpurun_out/final/prof_c5 $C > gpurun_out/final/ncu_full_c5.log 2>&1
echo "c5 full rc=$?"
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline"
$C4 > gpurun_out/final/plain_c4.log 2>&1 && ncu --set full --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 -o gpurun_out/final/prof_c4 $C4 > gpurun_out/final/ncu_c4.log 2>&1
echo "c4 full rc=$?"
C3="python bench.py --config 3 --mode batched --tile 64 --steps 1 --warmup 1 --no-cpu-baseline"
$C3 > gpurun_out/final/plain_c3b.log 2>&1 && ncu --set full --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 -o gpurun_out/final/prof_c3b $C3 > gpurun_out/final/ncu_c3b.log 2>&1
echo "c3b full rc=$?"
for c in c5 c4 c3b; do python profiles/ncu_summary.py gpurun_out/final/prof_$c.ncu-rep > gpurun_out/final/ncu_${c}_summary.txt 2>&1; done
ncu -i gpurun_out/final/prof_c5.ncu-rep --page details > gpurun_out/final/ncu_c5_details.txt 2>&1
rm -f gpurun_out/final/*.ncu-rep   # gpurun_out/ returns at most 64 MiB: the text pages are what is kept
ls -la gpurun_out/final/
