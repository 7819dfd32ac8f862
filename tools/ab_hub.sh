mkdir -p gpurun_out
for cfg in 1 2; do
 for i in 1 2; do
  for lib in paper_2412_10789_b200/libcpg.so tools/variants/libcpg_hub1024.so tools/variants/libcpg_hub512.so tools/variants/libcpg_hub256.so tools/variants/libcpg_hub128.so; do
    CPG_LIB_PATH=$lib python bench.py --no-cpu-baseline --config $cfg --mode batched 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$cfg', '$lib', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],4))"
  done
 done
done > gpurun_out/ab_hub.txt 2>&1
CPG_LIB_PATH=tools/variants/libcpg_hub128.so timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_hub128.log 2>&1
tail -2 gpurun_out/pytest_hub128.log >> gpurun_out/ab_hub.txt
