#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh NAME "-DFLAG=..."
set -e
name=$1; shift
out=tools/var/$name; mkdir -p $out/obj
for f in paper_2501_07778_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o $out/obj/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libqttb200.so $out/obj/*.o -cudart static
rm -rf $out/obj
