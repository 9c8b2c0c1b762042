set -x
timeout 600 python -m pytest tests/test_gpu_coupling.py tests/test_gpu_lu_int8.py -m gpu -q -s -k "coupling or componentwise" 2>&1 | grep -v "^$" | tail -30
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s 2>&1 | tail -12
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/p3_bench.json 2> gpurun_out/p3_bench.err; tail -c 6000 gpurun_out/p3_bench.json; tail -5 gpurun_out/p3_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/p3_ref.json 2>&1; tail -c 3000 gpurun_out/p3_ref.json
