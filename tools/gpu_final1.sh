#!/bin/bash
# Final round-2 check: bounds-checked build over the kernel paths and the GPU suite (full-size tests excluded),
# then every config's bench line with the refreshed ncu traffic.
bash tools/checked.sh gpurun_out/checked > gpurun_out/checked_summary.txt 2>&1
cat gpurun_out/checked_summary.txt
unset CPG_LIB_PATH
bash tools/bench_all.sh > gpurun_out/bench_all.txt 2>&1
cat gpurun_out/bench_all.txt
