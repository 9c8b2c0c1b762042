# round-2 (session 5): edge-case GPU tests
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider > gpurun_out/r30_edges.log 2>&1; echo "edges rc=$?"
tail -40 gpurun_out/r30_edges.log
