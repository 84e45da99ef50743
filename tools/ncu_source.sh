#!/bin/bash
# On the GPU box: ncu --set full of one launch of each kernel in $KLIST
# ("regex:skip" pairs, demangled names) in tools/profile_case.py, plus the
# per-line source page (SASS + CUDA correlation) as CSV.  Outputs under gpurun_out/$1/.
set -e
cd "$(dirname "$0")/.."
tag=${1:-src}; out=gpurun_out/$tag; mkdir -p $out
i=0
for ks in ${KLIST:-k_cell_sort_fixed:1 k_scatter<:2}; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$k" \
    --launch-skip $skip --launch-count 1 -o $out/k$i -f python tools/profile_case.py ${LOG2N:-28} 2 \
    > $out/k$i.log 2>&1 || echo "ncu $k failed"
  ncu -i $out/k$i.ncu-rep --page source --csv --print-source sass > $out/k${i}_sass.csv 2>/dev/null || true
  ncu -i $out/k$i.ncu-rep --page source --csv --print-source cuda > $out/k${i}_cuda.csv 2>/dev/null || true
  ncu -i $out/k$i.ncu-rep --page details --csv > $out/k${i}_details.csv 2>/dev/null || true
  rm -f $out/k$i.ncu-rep
  i=$((i+1))
done
ls -la $out
