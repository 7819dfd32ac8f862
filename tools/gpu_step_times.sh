mkdir -p gpurun_out/step_times
python -m pytest tests/test_gpu_sparse_steps.py -x -q 2>&1 | tail -3
python tools/step_times.py --config 5 --mode batched --M 0,2 --reps 1 > gpurun_out/step_times/c5_b.txt 2>&1
python tools/step_times.py --config 4 --mode batched --M 0,2 --reps 1 > gpurun_out/step_times/c4_b.txt 2>&1
