#!/bin/bash
# A/B timing of two kernel-variant selections (p2s_options.force bits) on one box:
#   tools/ab.sh <force_a> <force_b> [rounds] [workload]      e.g. tools/ab.sh 0 0x100 2 cfg3_512
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
R=${3:-2}
WL=${4:-cfg3_512}
for i in $(seq $R); do
  for F in "$1" "$2"; do
    timeout 600 python bench.py --workload "$WL" --extra none --steps 10 --warmup 3 --no-cpu-baseline --force "$F" 2>/dev/null |
      python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('force=$F', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), ' '.join(f'{k}={v[\"ms_per_launch\"]:.3f}' for k,v in s.items()), d['clocks']['sm_mhz'])"
  done
done
