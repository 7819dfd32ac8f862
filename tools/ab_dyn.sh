# Fused batched kernel: dynamic job claiming (default for B <= 16) vs static stride
# (CPG_DYN_JOBS=0), and against a reference build ($1) (GPU box)
head_lib=${1:-paper_2412_10789_b200/libcpg.so}
for spec in "1 16" "2 16" "2 64"; do
  set -- $spec
  for i in 1 2 3; do
    for dj in 1 0 head; do
      if [ $dj = head ]; then lib=$head_lib; e=1; else lib=paper_2412_10789_b200/libcpg.so; e=$dj; fi
      CPG_LIB_PATH=$lib CPG_DYN_JOBS=$e python bench.py --no-cpu-baseline --config $1 --mode batched --tile $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg$1 tile$2 dyn=$dj', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['launch_ms'],4))"
    done
  done
done
