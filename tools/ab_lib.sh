# A/B two library builds on one box: tools/ab_lib.sh <other.so> <bench args...>
other=$1; shift
for i in 1 2; do
  for lib in paper_2412_10789_b200/libcpg.so $other; do
    CPG_LIB_PATH=$lib python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', '$*', round(d['value'],1), round(d['roofline']['launch_ms'],4))"
  done
done
