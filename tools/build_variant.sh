#!/bin/bash
# Build a libkct variant with extra -D flags for A/B sweeps:
#   tools/build_variant.sh NAME -DKCT_FWD_WIN=0 ...   ->  build/libkct_NAME.so
# Load it with KCT_LIB_PATH=build/libkct_NAME.so.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/var_$name; mkdir -p "$out"
flags="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -diag-suppress 550"
objs=""
for s in projector solver fdk capi comm; do
  nvcc $flags "$@" -c "$root/paper_2509_08574_b200/csrc/$s.cu" -o "$out/$s.o" &
  objs="$objs $out/$s.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$root/build/libkct_$name.so" $objs -ldl
echo "$root/build/libkct_$name.so"
