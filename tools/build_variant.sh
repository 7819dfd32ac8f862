#!/bin/bash
# Build an A/B variant of libcpg.so with extra nvcc defines on every CUDA source:
#   tools/build_variant.sh <name> "-DCPG_GATHER_NA=1 ..."
# -> tools/variants/libcpg_<name>.so (git-ignored, travels to the GPU box).
# Compare on one box with tools/ab_lib.sh tools/variants/libcpg_<name>.so <bench args>.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
defs="$*"
python -m paper_2412_10789_b200._build >/dev/null
mkdir -p tools/variants build/variants/$name
objs=""
for src in paper_2412_10789_b200/csrc/*.cu; do
  b=$(basename $src)
  if [ "$b" = nccl_sym.cu ]; then objs="$objs build/cpg/$b.o"; continue; fi
  nvcc -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2412_10789_b200/csrc \
    -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr $defs \
    -c $src -o build/variants/$name/$b.o 2> build/variants/$name/$b.log &
  objs="$objs build/variants/$name/$b.o"
done
wait
objs="$objs $(ls build/cpg/*.cpp.o)"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/variants/libcpg_$name.so $objs -ldl -lpthread
echo tools/variants/libcpg_$name.so
