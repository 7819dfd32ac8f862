#!/bin/bash
# Final: GPU suite, refreshed ncu traffic of configs 4 and 3 (B = 64 thresholds changed), smoke.
mkdir -p gpurun_out/final2
python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/final2/pytest_gpu.txt
cat gpurun_out/final2/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.txt 2>&1; tail -1 gpurun_out/final2/smoke.txt
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline"
$C4 > gpurun_out/final2/plain_c4.log 2>&1 && ncu --set full --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 -o gpurun_out/final2/prof_c4 $C4 > gpurun_out/final2/ncu_c4.log 2>&1
C3="python bench.py --config 3 --mode batched --tile 64 --steps 1 --warmup 1 --no-cpu-baseline"
$C3 > gpurun_out/final2/plain_c3b.log 2>&1 && ncu --set full --clock-control none -k regex:"cheby_batch_(pieces|rows)" -s 6 -c 2 -o gpurun_out/final2/prof_c3b $C3 > gpurun_out/final2/ncu_c3b.log 2>&1
for c in c4 c3b; do python profiles/ncu_summary.py gpurun_out/final2/prof_$c.ncu-rep > gpurun_out/final2/ncu_${c}_summary.txt 2>&1; done
rm -f gpurun_out/final2/*.ncu-rep
grep -E "Kernel Name|gpu__time_duration|dram__bytes" gpurun_out/final2/ncu_c4_summary.txt gpurun_out/final2/ncu_c3b_summary.txt
