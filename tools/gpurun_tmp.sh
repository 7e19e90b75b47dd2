timeout 900 python -m pytest tests/test_gpu_knobs.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15
