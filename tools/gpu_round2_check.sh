#!/bin/bash
# Re-entry check: sparse-step tests, A/B of the sparse early steps, the whole GPU suite, default bench.
mkdir -p gpurun_out/r2check
python -m pytest tests/test_gpu_sparse_steps.py -x -q 2>&1 | tail -5 > gpurun_out/r2check/sparse_tests.txt
source tools/ab_sparse.sh
for M in 0 1 2 3; do CPG_SPARSE_STEPS=$M run c5_b16_M$M --steps 4 --warmup 3; done > gpurun_out/r2check/ab_c5.txt 2>&1
for M in 0 2 3 4; do CPG_SPARSE_STEPS=$M run c3_single_M$M --config 3 --steps 3 --warmup 3; done > gpurun_out/r2check/ab_c3.txt 2>&1
for M in 0 2; do CPG_SPARSE_STEPS=$M run c4_b64_M$M --config 4 --steps 3 --warmup 3; done > gpurun_out/r2check/ab_c4.txt 2>&1
for M in 0 2; do CPG_SPARSE_STEPS=$M run c1_M$M --config 1 --steps 5 --warmup 3; done > gpurun_out/r2check/ab_c1.txt 2>&1
for M in 0 2; do CPG_SPARSE_STEPS=$M run c2_M$M --config 2 --steps 5 --warmup 3; done > gpurun_out/r2check/ab_c2.txt 2>&1
python tools/step_times.py --config 5 --mode batched --M 0,2 --reps 1 > gpurun_out/r2check/step_times_c5.txt 2>&1
cat gpurun_out/r2check/ab_*.txt
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2check/pytest_gpu.txt
cat gpurun_out/r2check/pytest_gpu.txt gpurun_out/r2check/sparse_tests.txt
