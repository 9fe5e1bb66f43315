# S0 out-of-place sweeps vs L2 prefetch distance (all sweeps get the same distance)
for pf in 296 148 222 74 370 296; do
  QAOA_PF_DIST=$pf timeout 200 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pfs0_$pf.log 2>&1
  cp gpurun_out/pfs0_$pf.log gpurun_out/pfs0_${pf}_$(date +%s).log
done
