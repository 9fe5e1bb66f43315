#!/bin/bash
# ncu --set full (+ source) of one merged level-boundary sweep of an N=30 p=10
# fast run (run 2 of tools/prof_run.py: sweep 21 = launch control, 22 = S0,
# 23 = merged).  Tooling only; writes text exports into gpurun_out/.
R=${1:-r10}
ncu --set full --clock-control none --import-source on -k regex:sweep -s ${SKIP:-23} -c 1 \
    -o gpurun_out/merged_${R} python tools/prof_run.py 30 10 > gpurun_out/prof_merged_${R}.log 2>&1
ncu -i gpurun_out/merged_${R}.ncu-rep --page details --csv > gpurun_out/merged_details_${R}.csv
ncu -i gpurun_out/merged_${R}.ncu-rep --page raw --csv > gpurun_out/merged_raw_${R}.csv
ncu -i gpurun_out/merged_${R}.ncu-rep --page source --csv --print-source sass > gpurun_out/merged_source_${R}.csv
