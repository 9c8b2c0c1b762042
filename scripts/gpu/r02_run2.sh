# round-2: full GPU tests, c5 all shifts, c3 launch list, ncu --set full captures per kernel class
set -x
mkdir -p gpurun_out/ncu
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputests.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/r2_gputests.log
timeout 1500 python scripts/run_c5_shifts.py > gpurun_out/r2_c5_shifts.jsonl 2> gpurun_out/r2_c5_shifts.err; echo "c5 rc=$?"
tail -2 gpurun_out/r2_c5_shifts.jsonl
# launch list of one c3 bench step (cold-cache serialised per-launch times)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file gpurun_out/ncu/r2_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/ncu/r2_launch.log 2>&1; echo "launch list rc=$?"
NT="python scripts/ncu_target.py"
FULL="ncu --set full --clock-control none --import-source on"
# c3 full size (the bench workload): apply sweeps (after the 8 spike sweeps), INT8 update mid-LU
timeout 1200 $FULL -k regex:band_solve_kernel -s 8 -c 2 -o gpurun_out/ncu/r2_c3_apply $NT c3 1.0 nosolve 64 > gpurun_out/ncu/r2_c3_apply.log 2>&1; echo "c3 apply rc=$?"
timeout 1200 $FULL -k regex:lu_i8_gemm -s 20 -c 1 -o gpurun_out/ncu/r2_c3_lu_i8 $NT c3 1.0 nosolve 64 > gpurun_out/ncu/r2_c3_lu_i8.log 2>&1; echo "c3 lu_i8 rc=$?"
# the other kernel classes at c3 scale 0.75 (72^3, P=64; 17 GB of factors)
for k in lu_i8_slice lu_diag_kernel "lu_gemm_kernel<0" spmv multidot; do
  tag=$(echo "$k" | tr -cd 'a-z0-9_')
  timeout 900 $FULL -k "regex:$k" -s 3 -c 1 -o gpurun_out/ncu/r2_c3s_$tag $NT c3 0.75 solve 64 > gpurun_out/ncu/r2_c3s_$tag.log 2>&1; echo "$k rc=$?"
done
# spike sweeps: forward 48-column (first launch) and adjoint (second)
timeout 900 $FULL -k regex:band_solve_kernel -s 0 -c 2 -o gpurun_out/ncu/r2_c3s_spike $NT c3 0.75 nosolve 64 > gpurun_out/ncu/r2_c3s_spike.log 2>&1; echo "spike rc=$?"
# c5 structure (complex): LU update + sweeps
timeout 900 $FULL -k regex:lu_zgemm -s 10 -c 1 -o gpurun_out/ncu/r2_c5_zgemm $NT c5 0.5 nosolve > gpurun_out/ncu/r2_c5_zgemm.log 2>&1; echo "zgemm rc=$?"
timeout 900 $FULL -k regex:band_solve_z -s 4 -c 2 -o gpurun_out/ncu/r2_c5_zsolve $NT c5 0.5 nosolve > gpurun_out/ncu/r2_c5_zsolve.log 2>&1; echo "zsolve rc=$?"
ls -la gpurun_out/ncu
