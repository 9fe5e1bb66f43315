#!/bin/bash
# sweep_probe builds with extra -D definitions: tools/build_probe_defs.sh NAME "-DX=1 ..." [...]
# -> tools/ablib/sweep_probe_NAME.  A/B tooling only.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/ablib
F="-O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr -lcuda"
while [ $# -ge 2 ]; do
  nvcc $F $2 -I paper_2312_03019_b200/csrc tools/sweep_probe.cu paper_2312_03019_b200/csrc/qaoa_sweep.cu paper_2312_03019_b200/csrc/qaoa_sweep32.cu \
    paper_2312_03019_b200/csrc/qaoa_sweep_tma.cu paper_2312_03019_b200/csrc/qaoa_cut_table.cu \
    -o tools/ablib/sweep_probe_$1 &
  shift 2
done
wait
