# round-2: INT8 tile-per-CTA variants on c3 (quads) and c2 (pairs); bench
set -x
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r11_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-200 gpurun_out/r11_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 3 > gpurun_out/r11_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-200 gpurun_out/r11_lu_c2.jsonl
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r11_bench.json 2> gpurun_out/r11_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r11_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations','e2e']});print(d['kernel_ms_per_step']);print(d['roofline_lu_update']['frac'], d['roofline']['frac'], d['clocks'])"
