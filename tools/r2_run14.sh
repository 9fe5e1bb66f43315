S=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_full.log 2>&1; E=$(date +%s); echo "wall $((E-S)) s"; tail -c 2500 gpurun_out/r2_ref_full.log
