# Cost of the post-wait L1 invalidation on the paths without PDL benefit (CPG_PDL=0 everywhere).
for cfg in "5 --mode single --steps 3" "3"; do
  for rep in 1 2; do
    for v in r01 nofence cur; do
      case $v in r01|nofence) env="CPG_LIB_PATH=tools/variants/libcpg_$v.so" ;; cur) env="CPG_X=1" ;; esac
      env CPG_PDL=0 $env python bench.py --config $cfg --no-cpu-baseline --warmup 2 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg $v pdl0', round(d['value'],1), round(d['ms_per_step'],3), 'launch_ms', round(d['roofline']['launch_ms'],4))"
    done
  done
done
