set -x
timeout 600 python -m pytest tests/test_gpu_mixed.py -x -q -p no:cacheprovider 2>&1 | tail -8
