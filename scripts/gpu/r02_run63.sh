# round-2 (session 5): bulk tiles per CTA: c2 with 1 / 2 / 3, c3 with 2 / 4 / 8, c5-real-A / c4(0.25) with 2 / 8
set -x
for t in 1 2 3; do echo "c2 TPC $t"; LRS_VARIANT_CHILD=1 LRS_I8_TPC_RT=$t timeout 300 python scripts/lu_variants.py c2 1.0 8 6 2>&1 | cut -c1-200; done
for t in 2 4 8; do echo "c3 TPC $t"; LRS_VARIANT_CHILD=1 LRS_I8_TPC_RT=$t timeout 300 python scripts/lu_variants.py c3 1.0 64 3 2>&1 | cut -c1-200; done
for t in 2 4 8; do echo "c4 TPC $t"; LRS_VARIANT_CHILD=1 LRS_I8_TPC_RT=$t timeout 300 python scripts/lu_variants.py c4 0.25 64 4 2>&1 | cut -c1-200; done
