# round-2: clock64 role accounting of the INT8 bulk update (quads, c3 P=64, launch K=20; pairs c3 as well)
set -x
LRS_LIB=build/var_probe/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r19_probe_quad.log 2>&1; echo "quad rc=$?"
grep PROBE gpurun_out/r19_probe_quad.log | head -40
LRS_LU_QUAD=0 LRS_LIB=build/var_probe/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r19_probe_pair.log 2>&1; echo "pair rc=$?"
grep PROBE gpurun_out/r19_probe_pair.log | head -40
