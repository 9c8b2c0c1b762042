# round-2 (session 5): 4 bulk tiles per CTA by default -- INT8 / determinism tests, c2 and c3 bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_determinism.py tests/test_gpu_complex.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r64_bench_c2.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r64_bench_c2.json')); print({k:d[k] for k in ('value','t_lu_s','t_spikes_s','t_solve_s')}, d['e2e']['value'])"
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r64_bench_c3.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r64_bench_c3.json')); print({k:d[k] for k in ('value','t_lu_s','t_spikes_s','t_solve_s')}, d['e2e']['value'], d['clocks'])"
