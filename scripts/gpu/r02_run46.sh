# round-2 (session 5): final state -- GPU tests, smoke, default bench (with the CPU baseline leg), c2 bench
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r46_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r46_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r46_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r46_smoke.log
timeout 1500 python bench.py > gpurun_out/r46_bench.json 2> gpurun_out/r46_bench.err; echo "bench rc=$?"
cut -c1-1300 gpurun_out/r46_bench.json
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r46_bench_c2.json 2> gpurun_out/r46_bench_c2.err; echo "c2 rc=$?"
cut -c1-900 gpurun_out/r46_bench_c2.json
