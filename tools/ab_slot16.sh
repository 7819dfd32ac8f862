# fused batched kernel geometry at B = 16 (config 1) and the new B = 64 default (config 2)
for rep in 1 2; do
  for v in r01 0 84 64 44; do
    case $v in r01) env="CPG_LIB_PATH=tools/variants/libcpg_r01.so" ;; 0) env="CPG_X=1" ;; *) env="CPG_SLOT_CFG=$v" ;; esac
    env $env python bench.py --config 1 --no-cpu-baseline --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg 1 $v', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launch_ms', round(d['roofline']['launch_ms'],4))"
  done
  for v in r01 0; do
    case $v in r01) env="CPG_LIB_PATH=tools/variants/libcpg_r01.so" ;; 0) env="CPG_X=1" ;; esac
    env $env python bench.py --config 2 --no-cpu-baseline --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg 2 $v', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launch_ms', round(d['roofline']['launch_ms'],4))"
  done
done
