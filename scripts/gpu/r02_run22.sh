# round-2 re-entry (session 4): warp-wide MMA issue A/B (default vs build/var_nowi), full GPU suite, smoke, c3 bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lu_int8.py -q -p no:cacheprovider > gpurun_out/r22_i8tests.log 2>&1; echo "i8 tests rc=$?"
tail -2 gpurun_out/r22_i8tests.log
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r22_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-220 gpurun_out/r22_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 3 > gpurun_out/r22_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-220 gpurun_out/r22_lu_c2.jsonl
LRS_LIB=build/var_probewi/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r22_probe_quad.log 2>&1; echo "probe rc=$?"
grep PROBE gpurun_out/r22_probe_quad.log | head -12
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r22_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r22_gputests.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r22_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r22_smoke.log
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r22_bench.json 2> gpurun_out/r22_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r22_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations','e2e','gpu_launches']});print(d['kernel_ms_per_step']);print(d['roofline']['frac'], d['roofline_lu_update']['frac'], d['clocks'])"
