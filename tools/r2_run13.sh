bash tools/profile_round.sh r08 > gpurun_out/profile_r08.log 2>&1; echo rc=$?
ncu --set full --clock-control none -k regex:cut_table -c 1 -o gpurun_out/cut_full_r08 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/cut_full_r08.ncu-rep --page raw --csv > gpurun_out/cut_raw_r08.csv; rm -f gpurun_out/cut_full_r08.ncu-rep
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench2.log 2>&1; tail -c 3500 gpurun_out/r2_bench2.log
