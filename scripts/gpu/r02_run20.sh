# round-2: clock64 accounting of the 2-SM INT8 bulk update (pairs and quads, c3 P=64, launch K=20)
set -x
LRS_I8_2SM=1 LRS_LIB=build/var_probe/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r20_probe2_quad.log 2>&1; echo "quad rc=$?"
grep PROBE2 gpurun_out/r20_probe2_quad.log | head -20
LRS_I8_2SM=1 LRS_LU_QUAD=0 LRS_LIB=build/var_probe/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r20_probe2_pair.log 2>&1; echo "pair rc=$?"
grep PROBE2 gpurun_out/r20_probe2_pair.log | head -20
