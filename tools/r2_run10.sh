tools/ab_r2.sh 2>&1 | tee gpurun_out/r2_ab3.log | cut -c 1-330
