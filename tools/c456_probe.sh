cd /root/repo
for r in 1 2; do
for kind in "4 12 0x1c" "5 12 0x1c" "6 12 0x1c" "5 21 0x1c"; do
  set -- $kind
  for sw in 0 2; do
    echo "C=$1 q=$2 flags=$3 QAOA_SWEEP32=$sw: $(QAOA_SWEEP32=$sw tools/sweep_probe 30 200 3 custom $1 $2 $3)"
  done
done
done
A="QAOA_SWEEP32=1" B="QAOA_SWEEP32=2" ROUNDS=2 STEPS=4 BENCH_ARGS="--qubits 33 --graph er --levels 4" bash tools/ab_env.sh
