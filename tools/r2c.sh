timeout 120 python tools/trace_fwdpp.py 2>&1 | tail -6
S2_FWD_PP=1 timeout 600 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
for E in "S2_FWD_PP=0" "S2_FWD_PP=1"; do echo "== $E"; env $E timeout 120 python tools/perf_fwd.py 2>&1 | tail -1; done
done
