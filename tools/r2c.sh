for r in 1 2; do
for v in "" pr2 pr4; do
echo "== '$v' $(S2ATTN_VARIANT=$v timeout 120 python tools/perf_bwd.py --uniform 2>&1 | tail -1 | cut -c1-200)"
done
done
