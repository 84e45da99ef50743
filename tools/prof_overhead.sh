#!/bin/bash
# cProfile of tools/overhead.py (host overhead per sort at small n).
python -m cProfile -o /tmp/p.out tools/overhead.py ${1:-16} ${2:-200} && python -c "
import pstats; pstats.Stats('/tmp/p.out').sort_stats('tottime').print_stats(22)" 2>&1 | tail -34
