#!/bin/bash
# GPU round: pytest -m gpu, then bench with the bucket-major final sort on / off.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
for bm in 1 0; do AMS_FINAL_BM=$bm timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_bm$bm.json 2> gpurun_out/bench_bm$bm.err; echo bench$bm=$?; python -c "
import json;d=json.loads(open('gpurun_out/bench_bm$bm.json').read().strip().splitlines()[-1]);print($bm, d['ms_per_step'], d['verified'], d['final_sort_cells']);print({k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
