# round-2 (session 5): is the non-symmetric LU slower than in session 4 because of the code or the box?
# build/var_s4 = the library at commit 88e5913 (session 4's last), against the current library with LRS_LU_SYM=0
set -x
mkdir -p gpurun_out
for i in 1 2; do
LRS_VARIANT_CHILD=1 LRS_LU_SYM=0 timeout 600 python scripts/lu_variants.py c3 1.0 64 3 2>&1 | cut -c1-200
LRS_VARIANT_CHILD=1 LRS_LIB=build/var_s4/liblrspike_cuda.so timeout 600 python scripts/lu_variants.py c3 1.0 64 3 2>&1 | cut -c1-200
LRS_VARIANT_CHILD=1 LRS_LU_SYM=0 timeout 600 python scripts/lu_variants.py c2 1.0 8 5 2>&1 | cut -c1-200
LRS_VARIANT_CHILD=1 LRS_LIB=build/var_s4/liblrspike_cuda.so timeout 600 python scripts/lu_variants.py c2 1.0 8 5 2>&1 | cut -c1-200
done
