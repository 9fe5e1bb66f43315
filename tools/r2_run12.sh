for ld in 0 1 2; do for G in 2 8; do echo -n "ld=$ld "; QAOA_XCHG_LD=$ld python tools/shard_probe.py 30 $G 3 | tail -1; done; done 2>&1 | tee gpurun_out/r2_xchg_ld.log
