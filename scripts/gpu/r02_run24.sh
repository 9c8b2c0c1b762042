# round-2 (session 5, re-created container): state check -- GPU tests, smoke, default bench, reference arm
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r24_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r24_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r24_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r24_smoke.log
timeout 1200 python bench.py > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err; echo "bench rc=$?"
cut -c1-1500 gpurun_out/r24_bench.json
