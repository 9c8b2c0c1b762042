# round-2 checkpoint: full GPU suite, smoke, c3 bench (with CPU baseline), c2 bench, reference arm, c5 all 8 shifts
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r14_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r14_gputests.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r14_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r14_smoke.log
timeout 1500 python bench.py > gpurun_out/r14_bench.json 2> gpurun_out/r14_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r14_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations','e2e','gpu_launches']});print(d['kernel_ms_per_step']);print(d['roofline']['frac'], d['roofline_lu_update']['frac'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r14_bench_c2.json 2> gpurun_out/r14_bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r14_bench_ref.json 2> gpurun_out/r14_bench_ref.err; echo "ref rc=$?"
cut -c1-300 gpurun_out/r14_bench_ref.json
timeout 1500 python scripts/run_c5_shifts.py > gpurun_out/r14_c5_shifts.jsonl 2> gpurun_out/r14_c5_shifts.err; echo "c5 rc=$?"
tail -1 gpurun_out/r14_c5_shifts.jsonl
