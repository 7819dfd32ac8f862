# A/B run-time settings on one box, interleaved, R rounds:
#   R=2 tools/ab_env.sh "CPG_CB_MB=0 CPG_CB_MB=512 ..." <bench args...>
# (one setting per word, several variables joined by commas; "-" = none)
sets=$1; shift
for i in $(seq 1 ${R:-2}); do
  for kv in $sets; do
    if [ "$kv" = "-" ]; then e=""; else e=$(echo "$kv" | tr "," " "); fi
    env $e python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$kv', '$*', round(d['value'],1), round(d['roofline']['launch_ms'],4), d['clocks']['sm_mhz'])"
  done
done
