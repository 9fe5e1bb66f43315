#!/bin/bash
# Bench A/B of the 128 x 32 policy (QAOA_SWEEP32=0 off / 1 policy / 2 every
# supported sweep) at the BASELINE sizes and N=22 / 28 (C = 7 / 4 sets), plus
# per-kind probe times for C = 4..6 merged sweeps.  Tooling only.
cd "$(dirname "$0")/.."
tools/sweep_probe check 13 24 32 | grep -E "FAIL|check:" | tail -3
for kind in "3 12 0x1c" "4 12 0x1c" "5 12 0x1c" "6 12 0x1c" "7 12 0x1c" "5 12 0x4" "5 12 0x64"; do
  set -- $kind
  for sw in 0 2; do
    echo "C=$1 flags=$3 QAOA_SWEEP32=$sw: $(QAOA_SWEEP32=$sw tools/sweep_probe 30 200 3 custom $1 $2 $3)"
  done
done
A="QAOA_SWEEP32=0" B="QAOA_SWEEP32=1" ROUNDS=2 bash tools/ab_env.sh
A="QAOA_SWEEP32=0" B="QAOA_SWEEP32=1" ROUNDS=2 STEPS=4 BENCH_ARGS="--qubits 33 --graph er --levels 4" bash tools/ab_env.sh
A="QAOA_SWEEP32=1" B="QAOA_SWEEP32=2" ROUNDS=1 STEPS=4 BENCH_ARGS="--qubits 33 --graph er --levels 4" bash tools/ab_env.sh
A="QAOA_SWEEP32=0" B="QAOA_SWEEP32=1" ROUNDS=2 STEPS=20 BENCH_ARGS="--qubits 26 --levels 4" bash tools/ab_env.sh
A="QAOA_SWEEP32=0" B="QAOA_SWEEP32=1" ROUNDS=2 STEPS=40 BENCH_ARGS="--qubits 28 --levels 4" bash tools/ab_env.sh
A="QAOA_SWEEP32=0" B="QAOA_SWEEP32=1" ROUNDS=2 STEPS=50 BENCH_ARGS="--qubits 22 --levels 4" bash tools/ab_env.sh
