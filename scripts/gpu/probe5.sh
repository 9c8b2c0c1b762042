set -x
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py 2>&1 | tail -25
timeout 600 python -m pytest tests/test_gpu_cpp_api.py -m gpu -q -s 2>&1 | tail -30
bash scripts/gpu/sanitize.sh 2>&1
