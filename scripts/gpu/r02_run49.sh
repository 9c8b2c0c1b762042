# round-2 (session 5): Omega drawn into page-locked memory and uploaded on a copy stream under the LU -- all GPU tests, bench, c4 setup profile
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r49_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r49_gpu_tests.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r49_bench.json 2> gpurun_out/r49_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r49_bench.json'))
print({k:d[k] for k in ('value','t_factorize_s','t_lu_s','t_spikes_s','t_solve_s','iterations')}, d['e2e'])"
timeout 600 python scripts/dev/setup_profile.py c4 0.25 2>&1 | tail -1 | cut -c1-600
timeout 600 python bench.py --config c2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','t_lu_s','t_spikes_s','t_solve_s')}, d['e2e']['value'])"
