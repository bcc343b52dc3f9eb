#!/bin/bash
# Build an experimental variant of the library: tools/build_variant.sh NAME "-DSCAN_WARPS=24 ..."
# Output: build_var/libcompass_NAME.so (git-ignored; travels to the GPU box with gpurun).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build_var/$name; mkdir -p $out
for f in paper_2102_02440_b200/csrc/*.cu; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr $@ -I include -I paper_2102_02440_b200/csrc -c $f -o $out/$(basename $f).o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o build_var/libcompass_$name.so $out/*.o -lcudart_static
echo build_var/libcompass_$name.so
