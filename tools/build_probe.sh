#!/bin/bash
# Build tools/sweep_probe from the current csrc and (if present) the A/B base
# copy tools/ablib/base -> tools/ablib/sweep_probe_base.  Tooling only.
set -e
cd "$(dirname "$0")/.."
F="-O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr -lcuda"
nvcc $F -I paper_2312_03019_b200/csrc tools/sweep_probe.cu paper_2312_03019_b200/csrc/qaoa_sweep.cu paper_2312_03019_b200/csrc/qaoa_sweep32.cu \
  paper_2312_03019_b200/csrc/qaoa_sweep_tma.cu paper_2312_03019_b200/csrc/qaoa_cut_table.cu -o tools/sweep_probe &
if [ -d tools/ablib/base ]; then
  nvcc $F -I tools/ablib/base tools/sweep_probe.cu tools/ablib/base/qaoa_sweep.cu \
    tools/ablib/base/qaoa_sweep_tma.cu tools/ablib/base/qaoa_cut_table.cu -o tools/ablib/sweep_probe_base &
fi
wait
