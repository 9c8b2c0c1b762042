# round-2: full GPU suite after the SVD completion / iface / Krylov changes, 2-SM LU variants
# with CTA-scope remote arrives, c3 bench
set -x
mkdir -p gpurun_out/ncu
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r5_gputests.log | tail -20
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r5_lu_c3.jsonl 2>&1; echo "lu c3 rc=$?"
cut -c1-300 gpurun_out/r5_lu_c3.jsonl
LRS_I8_2SM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm2 -s 12 -c 1 -o gpurun_out/ncu/r5_c3s_lu_i8_2sm python scripts/ncu_target.py c3 0.75 nosolve 64 > gpurun_out/ncu/r5_2sm.log 2>&1; echo "2sm ncu rc=$?"
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r5_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations']});print(d['kernel_ms_per_step'])"
