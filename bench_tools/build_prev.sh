#!/bin/bash
# build build/libtttattn_prev.so from build/prev_csrc (a snapshot of an earlier csrc/, dev A/B only)
set -e
mkdir -p build/prev_obj
for f in build/prev_csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude -Ipaper_2603_18567_b200/csrc -c $f -o build/prev_obj/$(basename $f .cu).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/libtttattn_prev.so build/prev_obj/*.o
