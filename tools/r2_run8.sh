KS="0 16 4" tools/decomp_probe.sh 2>&1 | sed 's/^/gather /' | tee gpurun_out/r2_decomp3.log
PROBE_OM=1 KS="0" tools/decomp_probe.sh 2>&1 | sed 's/^/om /' | tee -a gpurun_out/r2_decomp3.log
