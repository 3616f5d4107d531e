timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_bwd_variants.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2 3; do
for E in "S2_X=0" "S2ATTN_VARIANT=epi0"; do echo "== $E"; env $E timeout 120 python tools/perf_bwd.py --uniform 2>&1 | tail -1; done
done
timeout 120 python tools/trace_dkv.py 8 dq 2>&1 | tail -3
