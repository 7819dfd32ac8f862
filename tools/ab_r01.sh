# A/B of the current libcpg against round 1's build (tools/variants/libcpg_r01.so) on the
# small batched configs, interleaved on one box.
for cfg in "1" "2"; do
  for rep in 1 2; do
    for v in r01 cur_nopdl cur; do
      case $v in
        r01) env="CPG_LIB_PATH=tools/variants/libcpg_r01.so" ;;
        cur_nopdl) env="CPG_PDL=0" ;;
        cur) env="" ;;
      esac
      env $env python bench.py --config $cfg --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $cfg $v', round(d['value'],1), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'launch_ms', round(r['launch_ms'],4), 'share', round(r.get('step_share_of_device_time',0),3), 'launches', d.get('gpu_launches'))"
    done
  done
done
