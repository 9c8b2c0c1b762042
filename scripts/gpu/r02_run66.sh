set -x
for t in 8 4 2 1; do echo "c2 TPC3 $t"; LRS_VARIANT_CHILD=1 LRS_I8_TPC3=$t timeout 300 python scripts/lu_variants.py c2 1.0 8 6 2>&1 | cut -c1-200; done
for t in 8 2; do echo "c3 TPC3 $t"; LRS_VARIANT_CHILD=1 LRS_I8_TPC3=$t timeout 300 python scripts/lu_variants.py c3 1.0 64 3 2>&1 | cut -c1-200; done
