#!/bin/bash
mkdir -p gpurun_out/r2final
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2final/pytest_gpu.txt
cat gpurun_out/r2final/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2final/smoke.txt 2>&1; tail -2 gpurun_out/r2final/smoke.txt
bash tools/bench_all.sh > gpurun_out/bench_all.txt 2>&1
cat gpurun_out/bench_all.txt
