# round-2 (session 5): symmetric bulk update variants -- no C prefetch, 16 / 4 tiles per CTA
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r37_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-200 gpurun_out/r37_lu_c3.jsonl
