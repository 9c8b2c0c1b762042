# round-2: quads vs pairs on c3 P=64 and c2; ncu of the quad update; fused SpMV-dot test
set -x
mkdir -p gpurun_out/ncu
timeout 1200 python -m pytest tests/test_gpu_spmv_dot.py tests/test_gpu_determinism.py tests/test_gpu_lu_int8.py -q -p no:cacheprovider > gpurun_out/r3_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r3_tests.log
timeout 120 python scripts/micro/read_bw.py > gpurun_out/r3_read_bw.json 2>&1; cat gpurun_out/r3_read_bw.json
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r3_lu_c3.jsonl 2>&1; echo "lu c3 rc=$?"
cat gpurun_out/r3_lu_c3.jsonl | cut -c1-400
timeout 600 python scripts/lu_variants.py c2 1.0 8 5 > gpurun_out/r3_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cat gpurun_out/r3_lu_c2.jsonl | cut -c1-400
LRS_LU_QUAD=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm -s 12 -c 1 -o gpurun_out/ncu/r3_c3s_lu_i8_quad python scripts/ncu_target.py c3 0.75 nosolve 64 > gpurun_out/ncu/r3_quad.log 2>&1; echo "quad ncu rc=$?"
LRS_I8_2SM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm2 -s 12 -c 1 -o gpurun_out/ncu/r3_c3s_lu_i8_2sm python scripts/ncu_target.py c3 0.75 nosolve 64 > gpurun_out/ncu/r3_2sm.log 2>&1; echo "2sm ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm_kernel -s 12 -c 1 -o gpurun_out/ncu/r3_c3s_lu_i8_pair python scripts/ncu_target.py c3 0.75 nosolve 64 > gpurun_out/ncu/r3_pair.log 2>&1; echo "pair ncu rc=$?"
