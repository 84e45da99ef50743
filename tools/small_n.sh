#!/bin/bash
# Timelines of the latency-bound shapes (config 1, config 5 ends): tools/small_n.sh TAG
cd "$(dirname "$0")/.."
out=gpurun_out/${1:-small}; mkdir -p $out
{
AMS_HOST_TRACE=1 python tools/timeline_case.py 20 16 16 0 16
AMS_HOST_TRACE=1 python tools/timeline_case.py 10 256 256 1
AMS_HOST_TRACE=1 python tools/timeline_case.py 16 256 256 1
AMS_HOST_TRACE=1 python tools/timeline_case.py 24 256 256 1
AMS_HOST_TRACE=1 python tools/timeline_case.py 10 256 8,32 1
AMS_HOST_TRACE=1 python tools/timeline_case.py 24 256 8,32 1
} > $out/timelines.txt 2>&1
tail -3 $out/timelines.txt
