# round-2: warp-wide MMA issue (elect.sync) in the INT8 update: probe + LU variants + INT8 tests
set -x
LRS_LIB=build/var_probewi/liblrspike_cuda.so timeout 600 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r21_probe_quad.log 2>&1; echo "probe rc=$?"
grep PROBE gpurun_out/r21_probe_quad.log | grep mma | head -6
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r21_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-220 gpurun_out/r21_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 3 > gpurun_out/r21_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-220 gpurun_out/r21_lu_c2.jsonl
timeout 900 python -m pytest tests/test_gpu_lu_int8.py -q -p no:cacheprovider > gpurun_out/r21_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r21_tests.log
