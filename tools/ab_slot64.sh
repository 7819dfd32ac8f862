# fused batched kernel geometry at B = 64 (config 2) with the mass check: CPG_SLOT_CFG = U*10 + CTAs/SM
for rep in 1 2; do
  for v in r01 0 64 44 83 63; do
    case $v in r01) env="CPG_LIB_PATH=tools/variants/libcpg_r01.so" ;; 0) env="CPG_X=1" ;; *) env="CPG_SLOT_CFG=$v" ;; esac
    env $env python bench.py --config 2 --no-cpu-baseline --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg 2 $v', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launch_ms', round(d['roofline']['launch_ms'],4), 'mass_err', d.get('mass_err_max'))"
  done
done
