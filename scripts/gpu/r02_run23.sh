# round-2 (session 4): one-pass 128x64 INT8 update (7 resident group accumulators) vs the two-pass kernel:
# INT8 tests on the variant, LU variants c3 / c2, clock64 probes of both at launch K=20
set -x
mkdir -p gpurun_out
LRS_LIB=build/var_onepass/liblrspike_cuda.so timeout 900 python -m pytest tests/test_gpu_lu_int8.py -q -x -p no:cacheprovider > gpurun_out/r23_i8tests_onepass.log 2>&1; echo "onepass i8 tests rc=$?"
tail -3 gpurun_out/r23_i8tests_onepass.log
timeout 900 python -m pytest tests/test_gpu_lu_int8.py -q -x -p no:cacheprovider > gpurun_out/r23_i8tests.log 2>&1; echo "i8 tests rc=$?"
tail -2 gpurun_out/r23_i8tests.log
LRS_LIB=build/var_probe20/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r23_probe_quad.log 2>&1; echo "probe rc=$?"
grep PROBE gpurun_out/r23_probe_quad.log | head -9
LRS_LIB=build/var_onepassprobe/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r23_probe_onepass.log 2>&1; echo "probe onepass rc=$?"
grep PROBE gpurun_out/r23_probe_onepass.log | head -9
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r23_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-220 gpurun_out/r23_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 3 > gpurun_out/r23_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-220 gpurun_out/r23_lu_c2.jsonl
