for r in 1 2; do
for v in old4 old3; do
echo "== variant '$v' $(S2ATTN_VARIANT=$v timeout 120 python tools/perf_fwd.py --n 131072 --h 32 --b 1 --v 16 --iters 5 2>&1 | tail -1)"
done
done
