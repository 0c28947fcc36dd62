#!/bin/bash
# Short bench of named workloads (TAG labels the lines): tools/wl.sh cfg4_1080p cfg5_4k ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for W in "$@"; do
  timeout 600 python bench.py --workload "$W" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null |
    python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('$W', '${TAG:-}', round(d['value'],1), ' '.join(f'{k}={v[\"ms_per_launch\"]:.3f}' for k,v in s.items()))"
done
