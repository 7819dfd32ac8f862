# Hub-partial combine: loads 8 (default) / 4 / 1 at a time (CPG_PARTIAL_UNROLL), same order of adds.
for cfg in "1" "2" "5 --steps 3" "1 --mode single"; do
  for rep in 1 2; do
    for v in un1 un4 cur; do
      case $v in un1|un4) env="CPG_LIB_PATH=tools/variants/libcpg_$v.so" ;; cur) env="CPG_X=1" ;; esac
      env $env python bench.py --config $cfg --no-cpu-baseline --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg $v', round(d['value'],1), round(d['ms_per_step'],3), 'launch_ms', round(d['roofline']['launch_ms'],4))"
    done
  done
done
