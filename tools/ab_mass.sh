# A/B of the batched mass-check implementations (CPG_MASS_MODE, step_kernels.cu) against
# round 1's build (no batched mass check): interleaved on one box.
# usage: bash tools/ab_mass.sh "<configs>" <steps>
cfgs=${1:-"1 2 4 5"}; steps=${2:-10}
for cfg in $cfgs; do
  for rep in 1 2; do
    for v in r01 mass0 mass2 cur; do
      case $v in
        r01|mass0|mass2) env="CPG_LIB_PATH=tools/variants/libcpg_$v.so" ;;
        cur) env="CPG_X=1" ;;
      esac
      env $env python bench.py --config $cfg --no-cpu-baseline --steps $steps --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg $v', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launch_ms', round(r['launch_ms'],4), 'mass_err', d.get('mass_err_max'))"
    done
  done
done
