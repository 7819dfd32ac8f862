# Round-2 refresh on one box: every config's bench line, the default headline line, the reference arm,
# then the ncu launch list of the default bench and one ncu --set full capture of the config-5 step kernels.
bash tools/bench_all.sh > gpurun_out/bench_all.txt 2>&1
cat gpurun_out/bench_all.txt
C="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$C > gpurun_out/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $C > gpurun_out/ncu_list.log 2>&1
echo "launch list rc=$?"
$C > gpurun_out/plain_c5b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cheby_batch_(pieces|rows)" -s 2 -c 2 -o gpurun_out/prof_c5 $C > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
