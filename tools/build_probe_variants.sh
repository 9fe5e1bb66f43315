#!/bin/bash
# sweep_probe builds with parts of the fused sweep compiled out (QB_SKIP bits,
# qaoa_tile.cuh): tools/ablib/sweep_probe_skip<K>.  Timing decomposition only.
set -e
cd "$(dirname "$0")/.."
F="-O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr -lcuda"
for k in "$@"; do
  nvcc $F -DQB_SKIP=$k -I paper_2312_03019_b200/csrc tools/sweep_probe.cu paper_2312_03019_b200/csrc/qaoa_sweep.cu paper_2312_03019_b200/csrc/qaoa_sweep32.cu \
    paper_2312_03019_b200/csrc/qaoa_sweep_tma.cu paper_2312_03019_b200/csrc/qaoa_cut_table.cu \
    -o tools/ablib/sweep_probe_skip$k &
done
wait
