#!/bin/bash
# Build the A/B base library tools/ablib/libqaoa_base.so from tools/ablib/base (tooling).
set -e
cd "$(dirname "$0")/ablib"
for f in base/*.cu; do
  nvcc -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -c $f -o obj/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libqaoa_base.so obj/*.o -lcudart_static -Xcompiler -fPIC
