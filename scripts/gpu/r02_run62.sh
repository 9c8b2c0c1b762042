# round-2 (session 5): bulk tiles per CTA at run time on c2 (quads): 8 (default), 4, 2, 16
set -x
for t in 8 4 2 16 8 4; do
echo "TPC $t"; LRS_VARIANT_CHILD=1 LRS_I8_TPC_RT=$t timeout 300 python scripts/lu_variants.py c2 1.0 8 6 2>&1 | cut -c1-260
done
