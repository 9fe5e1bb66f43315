#!/bin/bash
# 128 x 32 kernel for C = 3..7 and launch control: parity (1e-13 against the
# 256 x 16 flow, every set of n = 13..24), per-kind timings with (impl 3) and
# without (impl 30) it, then bench A/B of launch control and of N=33.  Tooling.
cd "$(dirname "$0")/.."
tools/sweep_probe check 13 24 32 | grep -E "FAIL|check:" | tail -5
for kind in "3 12 0x7 gen-S1" "3 21 0x7 gen-S2" "5 12 0x1c merged-C5" "5 12 0x64 last-C5" "6 12 0x1c merged-C6" "7 12 0x1c merged-C7"; do
  set -- $kind
  for impl in 30 3; do
    r=$(tools/sweep_probe 30 ${REPS:-200} $impl custom $1 $2 $3)
    echo "$4 impl=$impl: $r"
  done
done
A="QAOA_SWEEP32_GEN=0" B="QAOA_SWEEP32_GEN=1" ROUNDS=2 bash tools/ab_env.sh
A="QAOA_SWEEP32=0" B="QAOA_SWEEP32=1" ROUNDS=2 STEPS=4 BENCH_ARGS="--qubits 33 --graph er --levels 4" bash tools/ab_env.sh
