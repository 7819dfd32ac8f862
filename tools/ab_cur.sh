# current build vs round 1 (tools/variants/libcpg_r01.so), interleaved on one box.
# usage: bash tools/ab_cur.sh "<config args>;<config args>..." reps
IFS=';' read -ra cfgs <<< "${1:-1;2;4;3}"
reps=${2:-2}
for cfg in "${cfgs[@]}"; do
  for rep in $(seq $reps); do
    for v in r01 cur; do
      case $v in r01) env="CPG_LIB_PATH=tools/variants/libcpg_r01.so" ;; cur) env="CPG_X=1" ;; esac
      env $env python bench.py --config $cfg --no-cpu-baseline --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg $v', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launch_ms', round(d['roofline']['launch_ms'],4), 'mass_err', d.get('mass_err_max'))"
    done
  done
done
