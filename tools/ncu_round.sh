#!/bin/bash
# On the GPU box: launch list of one bench run + ncu --set full of the second
# sort's hot kernels (tools/profile_case.py).  Outputs under gpurun_out/$1/.
#   tools/ncu_round.sh TAG [log2n]
set -e
cd "$(dirname "$0")/.."
tag=${1:-prof}; log2n=${2:-28}
out=gpurun_out/$tag; mkdir -p $out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > $out/ncu_launches.log 2>&1 || echo "launch list failed"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-k_hist|k_scatter|k_cell_sort}" --launch-skip ${KSKIP:-8} --launch-count ${KCOUNT:-8} \
  -o $out/full -f python tools/profile_case.py $log2n 2 > $out/ncu_full.log 2>&1 || echo "full failed"
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null || true
ls -la $out
# gpurun copies back at most 64 MiB: keep the report only when it fits.
if [ -f $out/full.ncu-rep ] && [ $(stat -c %s $out/full.ncu-rep) -gt 50000000 ]; then
  rm -f $out/full.ncu-rep; echo "full.ncu-rep dropped (size); full_raw.csv kept"
fi
