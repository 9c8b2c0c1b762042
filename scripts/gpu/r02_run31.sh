# round-2 (session 5): INT8 epilogue with software-pipelined TMEM loads (LRS_I8_LDPIPE) -- tests, A/B against build/var_nopipe
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_determinism.py -x -q -p no:cacheprovider > gpurun_out/r31_i8tests.log 2>&1; echo "i8 tests rc=$?"
tail -4 gpurun_out/r31_i8tests.log
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r31_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-230 gpurun_out/r31_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 5 > gpurun_out/r31_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-230 gpurun_out/r31_lu_c2.jsonl
timeout 600 python scripts/lu_variants.py c5 1.0 16 2 > gpurun_out/r31_lu_c5.jsonl 2>&1; echo "lu c5 rc=$?"
cut -c1-230 gpurun_out/r31_lu_c5.jsonl
