tools/decomp_probe.sh 2>&1 | tee gpurun_out/r2_decomp.log
C=12 Q=0 FLAGS="0x4 0x105" KS="0 1 8 15" tools/decomp_probe.sh 2>&1 | tee -a gpurun_out/r2_decomp.log
