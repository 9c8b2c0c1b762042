# round-2 (session 5): c2 LU 0.18 s vs 0.15 s in session 4 -- warp-wide MMA issue loop A/B on c2 (build/var_nowarp), clocks
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
timeout 600 python scripts/lu_variants.py c2 1.0 8 5 > gpurun_out/r32_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-230 gpurun_out/r32_lu_c2.jsonl
