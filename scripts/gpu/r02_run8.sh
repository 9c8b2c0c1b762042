# round-2: fused L+U apply sweeps: fused test first, GPU suite, c3 bench, config sweep with clocks
set -x
timeout 900 python -m pytest tests/test_gpu_fused_sweeps.py -q -p no:cacheprovider > gpurun_out/r8_fused.log 2>&1; echo "fused rc=$?"
tail -3 gpurun_out/r8_fused.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r8_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r8_gputests.log | tail -20
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r8_bench.json 2> gpurun_out/r8_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r8_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations']});print(d['kernel_ms_per_step']);print(d['roofline']);print(d['clocks'])"
for c in "c1 1.0 0" "c2 1.0 0" "c3 1.0 8" "c4 0.25 64"; do timeout 600 python scripts/run_config.py $c >> gpurun_out/r8_configs.jsonl 2>> gpurun_out/r8_configs.err; done; echo "configs rc=$?"
cut -c1-400 gpurun_out/r8_configs.jsonl
