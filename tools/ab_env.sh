#!/bin/bash
# Interleaved A/B of bench.py lines under two environment settings (tooling):
#   A="QAOA_GEN_AUX=0" B="QAOA_GEN_AUX=1" ROUNDS=3 tools/ab_env.sh
cd "$(dirname "$0")/.."
for i in $(seq ${ROUNDS:-3}); do
  for side in A B; do
    envs=${!side}
    env $envs python bench.py --steps ${STEPS:-10} --warmup 3 --e2e-steps 0 --no-cpu-baseline \
        --no-symmetric-probe --no-cut-table ${BENCH_ARGS} 2>/dev/null | tail -1 | python3 -c "
import json,sys
d=json.loads(sys.stdin.read())
pk={k:round(v['avg_ms'],3) for k,v in d['roofline']['per_kind'].items()}
print('$side', round(d['value'],2), d['clocks']['sm_mhz'], pk)"
  done
done
