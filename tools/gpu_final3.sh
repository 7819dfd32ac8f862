#!/bin/bash
# Final round-2 run on one box: GPU suite, smoke, ncu launch list + full captures (configs 5, 4, 3 batched),
# profiles/ncu_traffic.json rebuilt from them, then every config's bench line.
mkdir -p gpurun_out/final3
python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/final3/pytest_gpu.txt
cat gpurun_out/final3/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/smoke.txt 2>&1; tail -1 gpurun_out/final3/smoke.txt
bash tools/refresh_r02_final.sh > gpurun_out/final3/refresh.log 2>&1
python tools/update_ncu_traffic.py gpurun_out/final "profiles/r02/ncu_final (final round-2 build, tools/refresh_r02_final.sh)"
cp profiles/ncu_traffic.json gpurun_out/final3/ncu_traffic.json
bash tools/bench_all.sh > gpurun_out/bench_all.txt 2>&1
cat gpurun_out/bench_all.txt
