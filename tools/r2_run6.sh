KS="0 4 16 32 48" tools/decomp_probe.sh 2>&1 | tee gpurun_out/r2_decomp2.log
