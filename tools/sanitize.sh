# compute-sanitizer memcheck / racecheck / synccheck over every kernel path (tools/sanitize_paths.py).
# Writes profiles/r02/sanitizer/<tool>_<path>.log
out=${1:-gpurun_out/sanitizer}
mkdir -p $out
for path in single single_split group fused16 fused64 split16 split64 loopback p2p_self measure topk; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_paths.py $path > $out/${tool}_${path}.log 2>&1
    echo "$tool $path rc=$? $(grep -h 'ERROR SUMMARY\|max_abs' $out/${tool}_${path}.log | tr '\n' ' ')"
  done
done
