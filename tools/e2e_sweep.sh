#!/bin/bash
# e2e (host-buffer) frames/s under fixed sub-batch sizes vs the default schedule: tools/e2e_sweep.sh 8 16 32 ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() { timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null |
  python -c "import json,sys; d=json.load(sys.stdin); print('$1', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"; }
run default
for s in "$@"; do P2S_HOST_SUB=$s run "sub=$s"; done
