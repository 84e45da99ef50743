#!/bin/bash
# On the GPU box: one compute-sanitizer tool over tools/paths_case.py (every
# device path at small sizes).  tools/sanitize.sh TOOL [TAG]   TOOL = memcheck | racecheck | synccheck | initcheck
cd "$(dirname "$0")/.."
tool=${1:-memcheck}; out=gpurun_out/${2:-san}; mkdir -p $out
python tools/paths_case.py > $out/plain.log 2>&1 || { echo "plain run failed"; tail -5 $out/plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/paths_case.py > $out/$tool.log 2>&1
echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok|Error|hazard" $out/$tool.log | tail -25
