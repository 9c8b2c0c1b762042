# round-2 (session 5): symmetric schedule on the DMMA two-step kinds (LRS_LU_I8=0) -- LU tests, c3 LU with INT8 off
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider 2>&1 | tail -5
LRS_VARIANT_CHILD=1 LRS_LU_I8=0 timeout 600 python scripts/lu_variants.py c3 1.0 64 2 2>&1 | cut -c1-300
LRS_VARIANT_CHILD=1 LRS_LU_I8=0 LRS_LU_SYM=0 timeout 600 python scripts/lu_variants.py c3 1.0 64 2 2>&1 | cut -c1-300
