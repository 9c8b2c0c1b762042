# round-2: 2-SM INT8 update (correctness + LU variants + ncu), the failing GPU tests, c5 all shifts
set -x
mkdir -p gpurun_out/ncu
timeout 1500 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_failures.py tests/test_gpu_spmv_dot.py tests/test_gpu_determinism.py "tests/test_gpu_fullsize.py" -q -p no:cacheprovider > gpurun_out/r4_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r4_tests.log | tail -20
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r4_lu_c3.jsonl 2>&1; echo "lu c3 rc=$?"
cut -c1-300 gpurun_out/r4_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 5 > gpurun_out/r4_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-300 gpurun_out/r4_lu_c2.jsonl
LRS_I8_2SM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm2 -s 12 -c 1 -o gpurun_out/ncu/r4_c3s_lu_i8_2sm python scripts/ncu_target.py c3 0.75 nosolve 64 > gpurun_out/ncu/r4_2sm.log 2>&1; echo "2sm ncu rc=$?"
LRS_I8_2SM=1 LRS_LU_QUAD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm2 -s 12 -c 1 -o gpurun_out/ncu/r4_c3s_lu_i8_2sm_quad python scripts/ncu_target.py c3 0.75 nosolve 64 > gpurun_out/ncu/r4_2sm_quad.log 2>&1; echo "2sm quad ncu rc=$?"
timeout 1500 python scripts/run_c5_shifts.py > gpurun_out/r4_c5_shifts.jsonl 2> gpurun_out/r4_c5_shifts.err; echo "c5 rc=$?"
cut -c1-250 gpurun_out/r4_c5_shifts.jsonl
