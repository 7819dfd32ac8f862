#!/bin/bash
# Finer A/B of the sparse early steps and per-step times with deeper masks.
mkdir -p gpurun_out/r2check
source tools/ab_sparse.sh
for M in 0 1 2; do CPG_SPARSE_STEPS=$M run c1_M$M --config 1 --steps 8 --warmup 4; done > gpurun_out/r2check/ab2_c1.txt 2>&1
for M in 0 1 2 3; do CPG_SPARSE_STEPS=$M run c2_M$M --config 2 --steps 8 --warmup 4; done > gpurun_out/r2check/ab2_c2.txt 2>&1
for M in 0 1 2 3; do CPG_SPARSE_STEPS=$M run c3b_M$M --config 3 --mode batched --steps 3 --warmup 3; done > gpurun_out/r2check/ab2_c3b.txt 2>&1
for M in 0 1 2 3; do CPG_SPARSE_STEPS=$M run c4_M$M --config 4 --steps 3 --warmup 3; done > gpurun_out/r2check/ab2_c4.txt 2>&1
for M in 0 1 2; do CPG_SPARSE_STEPS=$M run c5s_M$M --config 5 --mode single --steps 3 --warmup 3; done > gpurun_out/r2check/ab2_c5s.txt 2>&1
cat gpurun_out/r2check/ab2_*.txt
CPG_SPARSE_KERNEL=1 python tools/step_times.py --config 5 --mode batched --M 4 --reps 1 > gpurun_out/r2check/step_times_c5_M4_scan.txt 2>&1
CPG_SPARSE_KERNEL=0 python tools/step_times.py --config 5 --mode batched --M 4 --reps 1 > gpurun_out/r2check/step_times_c5_M4_masked.txt 2>&1
python tools/step_times.py --config 5 --mode single --M 0,3 --reps 1 > gpurun_out/r2check/step_times_c5_single.txt 2>&1
python tools/step_times.py --config 3 --mode single --M 0,3 --reps 1 > gpurun_out/r2check/step_times_c3_single.txt 2>&1
tail -4 gpurun_out/r2check/step_times_c5_M4_*.txt gpurun_out/r2check/step_times_c5_single.txt gpurun_out/r2check/step_times_c3_single.txt
