# round-2: GMRES with one host sync per Arnoldi step: GPU suite, c3 bench
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r18_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r18_gputests.log | tail -10
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r18_bench.json 2> gpurun_out/r18_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r18_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations','e2e','round_trips']});print(d['kernel_ms_per_step']);print(d['clocks'])"
timeout 900 python scripts/run_c5_shifts.py 1.0 0 > gpurun_out/r18_c5.jsonl 2> gpurun_out/r18_c5.err; echo "c5 rc=$?"
cut -c1-300 gpurun_out/r18_c5.jsonl
