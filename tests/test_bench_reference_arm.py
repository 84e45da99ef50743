"""bench.py's reference arm (CPU only): the oracle port on every host core,
one bounded-sample sort per worker process per step."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def test_cpu_port_rate_parallel_small():
    w = dict(bench.WORKLOADS["cfg2"], log2n=14, p=16, groups=(4, 4))
    rate, sample, ms = bench.cpu_port_rate_parallel(w, workers=2, steps=1, warmup=1)
    assert rate > 0 and ms > 0
    assert "2 worker processes x 1 timed sort(s)" in sample
