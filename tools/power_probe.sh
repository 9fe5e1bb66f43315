#!/bin/bash
# Power / clock of one sweep kind run back to back (~3 s): tools/power_probe.sh IMPL KIND [N]
# (kinds as in tools/sweep_probe.cu; prints ms per sweep, median SM MHz and W)
N=${3:-30}
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/pw_$$.log &
P=$!
sleep 0.5
${PROBE:-tools/sweep_probe} $N ${REPS:-400} $1 $2
kill $P
python3 - /tmp/pw_$$.log <<'PY'
import sys, statistics
rows=[l.split(",") for l in open(sys.argv[1]) if l.strip()]
sm=[float(r[0]) for r in rows]; pw=[float(r[1]) for r in rows]
hot=[(s,p) for s,p in zip(sm,pw) if p > 400]
if hot:
    print(f"  under load: SM {statistics.median([h[0] for h in hot]):.0f} MHz, {statistics.median([h[1] for h in hot]):.0f} W ({len(hot)} samples)")
PY
