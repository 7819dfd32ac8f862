# Bounds-checked build (tools/build_variant.sh checked -DCPG_CHECKED=1) over every kernel path and the
# GPU test suite: a CPG_CHECK violation traps the kernel (status != 0) and prints the index and bound.
out=${1:-gpurun_out/checked}
mkdir -p $out
export CPG_LIB_PATH=tools/variants/libcpg_checked.so
for path in single single_split group fused16 fused64 split16 split64 loopback p2p_self measure topk; do
  timeout 600 python tools/sanitize_paths.py $path > $out/path_${path}.log 2>&1
  echo "checked $path rc=$? $(grep -h 'max_abs\|CPG_CHECK' $out/path_${path}.log | head -3 | tr '\n' ' ')"
done
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > $out/pytest_gpu_checked.log 2>&1
echo "pytest (checked build) rc=$? $(tail -1 $out/pytest_gpu_checked.log)"
grep -h "CPG_CHECK" $out/*.log | head
