# round-2 (session 5): symmetric bulk update, column-major walk of the triangle (build/var_symcol) vs row-major
set -x
mkdir -p gpurun_out/ncu
LRS_LIB=build/var_symcol/liblrspike_cuda.so timeout 900 python -m pytest tests/test_gpu_lu_int8.py -k "symmetric" -x -q -p no:cacheprovider > gpurun_out/r44_symtests.log 2>&1; echo "sym tests rc=$?"
tail -3 gpurun_out/r44_symtests.log
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r44_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-200 gpurun_out/r44_lu_c3.jsonl
LRS_LIB=build/var_symcol/liblrspike_cuda.so timeout 900 ncu --set full --clock-control none -k regex:lu_i8_gemm_kernel -s 16 -c 1 -o gpurun_out/ncu/r44_c3_lu_i8_symcol python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/ncu/r44_i8.log 2>&1; echo "i8 rc=$?"
python scripts/ncu_summary.py gpurun_out/ncu/r44_c3_lu_i8_symcol.ncu-rep 2>&1 | head -12
