set -x
LRS_VARIANT_CHILD=1 timeout 600 python scripts/lu_variants.py c3 1.0 64 8 2>&1 | cut -c1-400
