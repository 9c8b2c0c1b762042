# round-2: x-prefetching multi-RHS sweeps, INT8 panel fit rule: GPU suite, c3 bench, ncu of the
# new / changed kernels, c5 shifts 0 and 3 (apply = complex 16-RHS sweeps)
set -x
mkdir -p gpurun_out/ncu
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r7_gputests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r7_gputests.log | tail -20
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r7_bench.json').read().strip().splitlines()[-1]);print({k:d[k] for k in ['value','t_lu_s','t_spikes_s','t_solve_s','iterations']});print(d['kernel_ms_per_step']);print(d['clocks'])"
NT="python scripts/ncu_target.py"
FULL="ncu --set full --clock-control none --import-source on"
timeout 900 $FULL -k regex:band_solve_kernel -s 0 -c 4 -o gpurun_out/ncu/r7_c3s_spike $NT c3 0.75 nosolve 64 > gpurun_out/ncu/r7_spike.log 2>&1; echo "spike rc=$?"
timeout 900 $FULL -k regex:lu_i8_gemm_kernel -s 20 -c 1 -o gpurun_out/ncu/r7_c3_lu_i8_quad $NT c3 1.0 nosolve 64 > gpurun_out/ncu/r7_quad.log 2>&1; echo "quad rc=$?"
timeout 900 $FULL -k regex:iface_dots1 -s 2 -c 1 -o gpurun_out/ncu/r7_c3s_iface $NT c3 0.75 nosolve 64 > gpurun_out/ncu/r7_iface.log 2>&1; echo "iface rc=$?"
timeout 900 $FULL -k regex:spmv_dot2 -s 2 -c 1 -o gpurun_out/ncu/r7_c2_spmvdot $NT c2 1.0 solve > gpurun_out/ncu/r7_spmvdot.log 2>&1; echo "spmvdot rc=$?"
timeout 900 $FULL -k regex:band_solve_z -s 8 -c 2 -o gpurun_out/ncu/r7_c5_zsolve $NT c5 0.5 nosolve > gpurun_out/ncu/r7_zsolve.log 2>&1; echo "zsolve rc=$?"
timeout 900 python scripts/run_c5_shifts.py 1.0 0 3 > gpurun_out/r7_c5_shifts.jsonl 2> gpurun_out/r7_c5_shifts.err; echo "c5 rc=$?"
cut -c1-300 gpurun_out/r7_c5_shifts.jsonl
