# round-2: auto quads + 512-row Krylov chunks: full GPU suite, c3 bench (with CPU baseline), c2 bench
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r6_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r6_gputests.log | tail -20
timeout 1500 python bench.py > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r6_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations','e2e']});print(d['kernel_ms_per_step']);print(d['roofline_lu_update']['frac'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r6_bench_c2.json 2> gpurun_out/r6_bench_c2.err; echo "bench c2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r6_bench_c2.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations']});print(d['kernel_ms_per_step'])"
