#!/bin/bash
# A/B of library variants on cfg2: tools/ab_libs.sh name1 name2 ... ("main" = the in-tree build)
cd "$(dirname "$0")/.."
for v in "$@"; do
  for rep in 1 2; do
    lib=paper_1410_6754_b200/lib/libams_b200.so; [ "$v" != main ] && lib=tools/abl/$v.so
    AMS_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweeps \
      ${WORKLOAD:+--workload $WORKLOAD} 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', round(d['ms_per_step'],3), d['verified']['sorted_and_checksum'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if v['ms_per_step']>0.05})"
  done
done
