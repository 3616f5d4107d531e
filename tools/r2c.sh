timeout 300 python tools/perf_units.py 2>&1 | tail -4
