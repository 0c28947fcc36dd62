#!/bin/bash
# A/B of two in-tree builds including the end-to-end (host buffers) number: tools/ab_e2e.sh libA.so libB.so [rounds]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for i in $(seq ${3:-1}); do
  for L in "$1" "$2"; do
    P2S_LIB_NAME=$L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('$L', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), ' '.join(f'{k}={v[\"ms_per_launch\"]:.3f}' for k,v in s.items()), d['clocks']['sm_mhz'])"
  done
done
