#!/bin/bash
# Device + e2e numbers of named workloads: tools/wl_e2e.sh cfg3_512 cfg4_1080p ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for W in "$@"; do
  timeout 900 python bench.py --workload "$W" --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('$W', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), ' '.join(f'{k}={v[\"ms_per_launch\"]:.3f}' for k,v in s.items()), 'blur_frac', round(d['roofline']['frac'],3))"
done
