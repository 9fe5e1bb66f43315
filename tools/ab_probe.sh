#!/bin/bash
# Interleaved A/B of sweep_probe builds (tools/ablib/sweep_probe_<V>) on sweep
# kinds "C q FLAGS name", with SM clock / power under load.  Tooling only.
#   VARIANTS="a b" KINDS="3 12 0x1c merged-S1;3 21 0x1c merged-S2" tools/ab_probe.sh
cd "$(dirname "$0")/.."
IFS=';' read -ra KL <<< "${KINDS:-3 12 0x1c merged-S1;3 21 0x1c merged-S2}"
for round in $(seq ${ROUNDS:-2}); do
for kind in "${KL[@]}"; do
  set -- $kind
  for vv in ${VARIANTS}; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/ab.log &
    P=$!
    sleep 0.3
    r=$(tools/ablib/sweep_probe_$vv 30 ${REPS:-200} ${IMPL:-3} custom $1 $2 $3)
    kill $P
    clk=$(python3 -c "
import statistics
rows=[l.split(',') for l in open('/tmp/ab.log') if l.strip()]
hot=[(float(a),float(b)) for a,b in rows if float(b)>400]
print(f'{statistics.median([h[0] for h in hot]):.0f} MHz {statistics.median([h[1] for h in hot]):.0f} W' if hot else 'idle')")
    echo "$4 $vv: $r | $clk"
  done
done
done
