# evict_first streams in the batched kernels (tools/variants/libcpg_streamef.so, -DCPG_STREAM_EF=1)
# against the default build, interleaved; then the hot-prefix budget under it on config 5.
for cfg in "5" "4" "3 --mode batched --tile 64" "2" "1"; do
  for rep in 1 2; do
    for v in cur streamef; do
      case $v in streamef) env="CPG_LIB_PATH=tools/variants/libcpg_streamef.so" ;; cur) env="CPG_X=1" ;; esac
      env $env python bench.py --config $cfg --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg $v', round(d['value'],1), round(d['ms_per_step'],2), 'launch_ms', round(d['roofline']['launch_ms'],3), 'mass', d['mass_err_max'])"
    done
  done
done
for hot in 32 96 126; do
  CPG_HOT_MB=$hot CPG_LIB_PATH=tools/variants/libcpg_streamef.so python bench.py --config 5 --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg 5 streamef hot=$hot', round(d['value'],1), round(d['ms_per_step'],2))"
done
