set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_complex.py -x -q -p no:cacheprovider 2>&1 | tail -3
