# round-2 (session 5): quads from 40 tiles per SM (c2 takes quads) -- c2 tests + bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_lu_int8.py -x -q -p no:cacheprovider > gpurun_out/r35_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r35_tests.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r35_bench_c2.json 2> gpurun_out/r35_bench_c2.err; echo "c2 rc=$?"
cut -c1-1100 gpurun_out/r35_bench_c2.json
