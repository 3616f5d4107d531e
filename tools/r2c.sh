timeout 900 python -m pytest tests/test_gpu_fwd.py -m gpu -q -x -p no:cacheprovider -k "f32" 2>&1 | tail -3
