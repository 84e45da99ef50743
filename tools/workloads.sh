#!/bin/bash
# Bench every single-GPU workload once (short runs): tools/workloads.sh [steps]
cd "$(dirname "$0")/.."
st=${1:-3}
for w in ${WL:-cfg1 cfg2 cfg3 cfg4a cfg4b cfg4c cfg4d}; do
  timeout 600 python bench.py --workload $w --steps $st --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$w', round(d['ms_per_step'],3), f\"{d['value']/1e9:.2f} Gkeys/s\", d.get('verified'), d.get('final_sort_cells'))" || echo "$w failed"
done
