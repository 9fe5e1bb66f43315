#!/bin/bash
# A/B of the current build (B) against tools/ablib/libqaoa_base.so (A) in one box session.
cd "$(dirname "$0")/.."
for i in 1 2 3; do
  QB_ITERS=${ITERS:-10} QAOA_B200_LIB=$PWD/tools/ablib/libqaoa_base.so python tools/quick_bench.py ${CFG:-30:10} | grep '"exact": false' | sed 's/^/A /'
  QB_ITERS=${ITERS:-10} python tools/quick_bench.py ${CFG:-30:10} | grep '"exact": false' | sed 's/^/B /'
done
