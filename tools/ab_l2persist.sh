# L2 persisting set-aside (CPG_L2_PERSIST_MB) x hot-prefix budget (CPG_HOT_MB) on configs 5 and 4.
for cfg in 5 4; do
  for v in "none 64" "64 64" "126 64" "126 96" "126 126" "none 64"; do
    set -- $v
    if [ $1 = none ]; then pe=""; else pe="CPG_L2_PERSIST_MB=$1"; fi
    env $pe CPG_HOT_MB=$2 python bench.py --config $cfg --no-cpu-baseline --steps 3 --warmup 3 2>gpurun_out/l2p.err | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $cfg persist=$1 hot=$2', round(d['value'],1), round(d['ms_per_step'],2), 'launch_ms', round(d['roofline']['launch_ms'],3))"
    grep "set-aside" gpurun_out/l2p.err | head -1
  done
done
