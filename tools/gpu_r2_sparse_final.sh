#!/bin/bash
# After the sparse-step defaults: sparse tests, per-step times, then every config's bench line.
mkdir -p gpurun_out/r2check
python -m pytest tests/test_gpu_sparse_steps.py -x -q 2>&1 | tail -5 > gpurun_out/r2check/sparse_tests2.txt
cat gpurun_out/r2check/sparse_tests2.txt
python tools/step_times.py --config 5 --mode batched --M 2 --reps 1 2>&1 | grep -E "step ms|total" | cut -c1-200 > gpurun_out/r2check/step_times_c5_fill2.txt
cat gpurun_out/r2check/step_times_c5_fill2.txt
bash tools/bench_all.sh > gpurun_out/bench_all.txt 2>&1
cat gpurun_out/bench_all.txt
