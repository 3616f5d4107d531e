timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/perf_bwd.py --uniform 2>&1 | tail -2
