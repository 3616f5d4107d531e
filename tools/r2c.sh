timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fullsize.py -m gpu -x -q -k "decode or cfg4" 2>&1 | tail -2
for r in 1 2 3; do
echo "pdl   $(timeout 200 python tools/perf_decode.py 2>&1 | tail -1)"
echo "nopdl $(S2_PDL=0 timeout 200 python tools/perf_decode.py 2>&1 | tail -1)"
done
