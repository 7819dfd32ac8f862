# Fused batched kernel: rows per job claim (CPG_CLAIM_ROWS builds) vs the static stride (GPU box)
for spec in "1 16" "2 16" "2 64"; do
  set -- $spec
  for i in 1 2; do
    for arm in claim4 claim8 claim16 static; do
      if [ $arm = static ]; then lib=tools/variants/libcpg_claim4.so; e=0; else lib=tools/variants/libcpg_$arm.so; e=1; fi
      CPG_LIB_PATH=$lib CPG_DYN_JOBS=$e python bench.py --no-cpu-baseline --config $1 --mode batched --tile $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$1 tile$2 $arm', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],4))"
    done
  done
done
