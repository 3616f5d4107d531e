S2ATTN_VARIANT=split4 timeout 600 python -m pytest tests/test_gpu_bwd_simt.py -m gpu -q 2>&1 | tail -1
for r in 1 2; do
for v in "" split4 split8; do
echo "== '$v' $(S2ATTN_VARIANT=$v timeout 120 python tools/perf_bwd_simt.py 2>&1 | tail -1)"
echo "== '$v' $(S2ATTN_VARIANT=$v timeout 120 python tools/perf_bwd_simt.py --d 128 --n 8192 2>&1 | tail -1)"
done
done
