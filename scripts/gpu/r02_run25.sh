# round-2 (session 5): symmetric LU schedule (lower trailing tiles + mirrored U panels) -- INT8 / fullsize tests, bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu_int8.py -x -q -p no:cacheprovider > gpurun_out/r25_i8tests.log 2>&1; echo "i8 tests rc=$?"
tail -15 gpurun_out/r25_i8tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -x -q -p no:cacheprovider > gpurun_out/r25_fullsize.log 2>&1; echo "fullsize rc=$?"
tail -8 gpurun_out/r25_fullsize.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r25_bench.json 2> gpurun_out/r25_bench.err; echo "bench rc=$?"
cut -c1-1200 gpurun_out/r25_bench.json
LRS_LU_SYM=0 timeout 1200 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/r25_bench_nosym.json 2> gpurun_out/r25_bench_nosym.err; echo "bench nosym rc=$?"
cut -c1-900 gpurun_out/r25_bench_nosym.json
