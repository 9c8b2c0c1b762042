set -x
for t in 8 4 2; do echo "c2 pairs TPC $t"; LRS_VARIANT_CHILD=1 LRS_LU_QUAD=0 LRS_I8_TPC_RT=$t timeout 300 python scripts/lu_variants.py c2 1.0 8 6 2>&1 | cut -c1-200; done
echo "c2 default"; LRS_VARIANT_CHILD=1 timeout 300 python scripts/lu_variants.py c2 1.0 8 6 2>&1 | cut -c1-200
