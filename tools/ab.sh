#!/bin/bash
# A/B the default library against variants: tools/ab.sh [variant ...] (names under tools/abl/)
cd "$(dirname "$0")/.."
for v in default "$@"; do
  if [ "$v" = default ]; then unset AMS_LIB; else export AMS_LIB=$PWD/tools/abl/$v.so; fi
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['kernels']
print('$v', round(d['ms_per_step'],3), ' '.join(f'{n}={v[\"ms_per_step\"]:.3f}' for n,v in k.items() if v['ms_per_step']>0.05), d.get('verified'))"
done
