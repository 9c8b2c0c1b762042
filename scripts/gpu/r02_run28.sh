# round-2 (session 5): symmetric blocks -- adjoint spike solves on the forward sweeps; all GPU tests + c3 bench
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r28_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -6 gpurun_out/r28_gpu_tests.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r28_bench.json 2> gpurun_out/r28_bench.err; echo "bench rc=$?"
cut -c1-1200 gpurun_out/r28_bench.json
