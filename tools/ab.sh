#!/bin/bash
# A/B timing of two builds of the engine in ONE gpurun call (box noise cancels):
#   tools/ab.sh <libA.so> <libB.so> [n:p ...]   (run under gpurun)
A=$1; B=$2; shift 2
for i in 1 2 3; do
  QAOA_B200_LIB=$A python tools/quick_bench.py "$@" | sed "s/^/A /" | grep '"exact": false'
  QAOA_B200_LIB=$B python tools/quick_bench.py "$@" | sed "s/^/B /" | grep '"exact": false'
done
