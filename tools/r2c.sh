timeout 900 python -m pytest tests/test_gpu_bwd_variants.py -m gpu -x -q 2>&1 | tail -2
S2_PREP_FUSED=1 timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -m gpu -x -q -k "not f32" 2>&1 | tail -2
for r in 1 2; do
echo "prep  $(timeout 120 python tools/perf_bwd.py --uniform 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-260)"
echo "fused $(S2_PREP_FUSED=1 timeout 120 python tools/perf_bwd.py --uniform 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-260)"
done
echo "cfg2 prep  $(timeout 120 python tools/perf_bwd.py --uniform --n 8192 --b 4 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-260)"
echo "cfg2 fused $(S2_PREP_FUSED=1 timeout 120 python tools/perf_bwd.py --uniform --n 8192 --b 4 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-260)"
