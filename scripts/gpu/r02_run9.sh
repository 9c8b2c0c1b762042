# round-2: interface setup tiling (GPU suite), bench with the fused-sweep roofline, LU cost split
# (LRS_LU_SKIP variants: bulk only / critical stream only), ncu of the fused sweep launch
set -x
mkdir -p gpurun_out/ncu
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r9_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r9_gputests.log | tail -20
timeout 1500 python bench.py > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r9_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations','e2e']});print(d['kernel_ms_per_step']);print(d['roofline']);print(d['roofline_lu_update']['frac']);print(d['clocks'])"
timeout 1200 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r9_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-260 gpurun_out/r9_lu_c3.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_solve_lu1 -s 0 -c 1 -o gpurun_out/ncu/r9_c3_apply_fused python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/ncu/r9_apply.log 2>&1; echo "apply ncu rc=$?"
