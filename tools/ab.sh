#!/bin/bash
# A/B timing of alternative in-tree builds on one box: tools/ab.sh libA.so libB.so [rounds]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
R=${3:-2}
for i in $(seq $R); do
  for L in "$1" "$2"; do
    P2S_LIB_NAME=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('$L', round(d['value'],1), ' '.join(f'{k}={v[\"ms_per_launch\"]:.3f}' for k,v in s.items()), d['clocks']['sm_mhz'])"
  done
done
