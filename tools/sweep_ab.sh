#!/bin/bash
# Same-box A/B of library variants on the config-5 sweep and config 1 (host-bound
# sizes vary from box to box): tools/sweep_ab.sh name1 name2 ... ("main" = in-tree)
cd "$(dirname "$0")/.."
for v in "$@" "$@"; do
  lib=paper_1410_6754_b200/lib/libams_b200.so; [ "$v" != main ] && lib=tools/abl/$v.so
  AMS_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
s=d['sweeps']
print('$v', round(d['ms_per_step'],3), 'rank', round(d['kernels']['sample_rank']['ms_per_step'],3), 'cfg1', round(s['cfg1']['ms_per_step'],3), round(s['cfg1_device_sampling']['ms_per_step'],3), 'k1', [round(r['ms_per_step'],2) for r in s['cfg5']['k1']], 'k2', [round(r['ms_per_step'],2) for r in s['cfg5']['k2']], 'k2dev', [round(r['ms_per_step'],2) for r in s['cfg5_device_sampling']['k2']])"
done
