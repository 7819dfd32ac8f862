# A/B several library builds on one box, interleaved, R rounds:
#   R=2 tools/ab_multi.sh "libA.so libB.so ..." <bench args...>
libs=$1; shift
for i in $(seq 1 ${R:-2}); do
  for lib in paper_2412_10789_b200/libcpg.so $libs; do
    CPG_LIB_PATH=$lib python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', '$*', round(d['value'],1), round(d['roofline']['launch_ms'],4), d['clocks']['sm_mhz'])"
  done
done
