#!/bin/bash
# A/B the default library under environment settings: tools/ab_env.sh "VAR=a" "VAR=b" ...
cd "$(dirname "$0")/.."
for v in "" "$@"; do
  env $v python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['kernels']
print('[$v]', round(d['ms_per_step'],3), ' '.join(f'{n}={v[\"ms_per_step\"]:.3f}' for n,v in k.items() if v['ms_per_step']>0.05), d.get('verified'), d.get('final_sort_cells'))"
done
