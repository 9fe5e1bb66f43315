#!/bin/bash
# C = 4..6 merged sweeps: 256 x 16 (QAOA_SWEEP32=0) against 128 x 32 at 3 CTAs
# per SM (probe build S32_MINB=3, QAOA_SWEEP32=2).  Tooling only.
cd "$(dirname "$0")/.."
for r in 1 2; do
for kind in "4 12 0x1c" "5 12 0x1c" "6 12 0x1c" "5 21 0x1c" "7 12 0x1c"; do
  set -- $kind
  echo "C=$1 q=$2 256x16: $(QAOA_SWEEP32=0 tools/sweep_probe 30 200 3 custom $1 $2 $3)"
  echo "C=$1 q=$2 128x32 m3: $(QAOA_SWEEP32=2 tools/ablib/sweep_probe_m3 30 200 3 custom $1 $2 $3)"
done
done
