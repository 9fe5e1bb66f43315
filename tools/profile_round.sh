#!/bin/bash
# Profiling recipe for one round (run under gpurun, 1 GPU; never multi-rank):
#   1. launch list of the bench command (cold-cache, serialised per-launch times)
#   2. `ncu --set full` of one sweep of each kind from one fused N=30 p=10 run
# Summaries are written as text into gpurun_out/ (the .ncu-rep stays small).
set -e
R=${1:-r01}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 200 --csv --log-file gpurun_out/launches_${R}.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-symmetric-probe > gpurun_out/bench_under_ncu_${R}.log 2>&1
# run 2 of tools/prof_run.py 30 10: sweeps 21..41 = gen (TMA in/out), S0 (one tile per CTA +
# L2 prefetch), merged top set (TMA-fed), S0, merged S1 (one tile per CTA + prefetch)
ncu --set full --clock-control none --import-source on -k regex:sweep -s 21 -c 5 \
    -o gpurun_out/sweep_full_${R} python tools/prof_run.py 30 10 > gpurun_out/prof_${R}.log 2>&1
ncu -i gpurun_out/sweep_full_${R}.ncu-rep --page details --csv > gpurun_out/sweep_details_${R}.csv
ncu -i gpurun_out/sweep_full_${R}.ncu-rep --page raw --csv > gpurun_out/sweep_raw_${R}.csv
ncu -i gpurun_out/sweep_full_${R}.ncu-rep --page source --csv --print-source sass > gpurun_out/sweep_source_${R}.csv
rm -f gpurun_out/sweep_full_${R}.ncu-rep
# symmetric half state (N=30 p=10): run 2's launch-control, mirror low-set and merged sweeps
ncu --set full --clock-control none --import-source on -k regex:sweep -s 21 -c 3 \
    -o gpurun_out/sym_full_${R} python tools/prof_sym.py 30 10 > gpurun_out/prof_sym_${R}.log 2>&1
ncu -i gpurun_out/sym_full_${R}.ncu-rep --page details --csv > gpurun_out/sym_details_${R}.csv
ncu -i gpurun_out/sym_full_${R}.ncu-rep --page raw --csv > gpurun_out/sym_raw_${R}.csv
rm -f gpurun_out/sym_full_${R}.ncu-rep
