timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_edges.py tests/test_gpu_fuzz.py tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2 3; do
for E in "S2_X=0" "S2ATTN_VARIANT=epi0" "S2ATTN_VARIANT=epi0n3"; do echo "== $E"; env $E timeout 120 python tools/perf_fwd.py 2>&1 | tail -1; done
done
timeout 120 python tools/trace_fwd.py 2>&1 | tail -2
