#!/bin/bash
# Round-end GPU evidence: tests, smoke, workloads, bench (cfg2), reference arm,
# then the launch list + ncu full set of the hot kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/${TAG:-final}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG:-final}/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG:-final}/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-final}/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG:-final}/smoke.log
timeout 600 python bench.py > gpurun_out/${TAG:-final}/bench.json 2> gpurun_out/${TAG:-final}/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG:-final}/bench_ref.json 2>&1; echo "ref rc=$?"
bash tools/workloads.sh 3 > gpurun_out/${TAG:-final}/workloads.txt 2>&1
bash tools/ncu_round.sh ${TAG:-final} 28 > /dev/null 2>&1; echo "ncu done"
