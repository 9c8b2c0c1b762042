# round-2 evidence: ncu of the complex INT8 update (c5) and the quad look-ahead pair update (c3),
# launch list of one c3 bench step
set -x
mkdir -p gpurun_out/ncu
NT="python scripts/ncu_target.py"
FULL="ncu --set full --clock-control none --import-source on"
timeout 900 $FULL -k regex:lu_i8_gemm_kernel -s 20 -c 1 -o gpurun_out/ncu/r16_c5_lu_i8_z $NT c5 1.0 nosolve > gpurun_out/ncu/r16_z.log 2>&1; echo "z rc=$?"
timeout 900 $FULL -k regex:lu_i8_slice_z -s 20 -c 1 -o gpurun_out/ncu/r16_c5_slice_z $NT c5 1.0 nosolve > gpurun_out/ncu/r16_sz.log 2>&1; echo "sz rc=$?"
timeout 900 $FULL -k regex:lu_i8_slice_kernel -s 20 -c 2 -o gpurun_out/ncu/r16_c3_slice $NT c3 1.0 nosolve 64 > gpurun_out/ncu/r16_s.log 2>&1; echo "s rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/ncu/r16_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu/r16_launch.log 2>&1; echo "launch rc=$?"
