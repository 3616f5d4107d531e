timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_selftest.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
