#!/bin/bash
# Config sweep for DESIGN.md section 7 (one B200): c1, c2, c3 (P=8, 64), c4 at scale 0.25,
# c5 one shift; then the bench under torchrun with one rank (the NCCL adapter path).
out=${1:-gpurun_out/configs.jsonl}
: > "$out"
for args in "c1 1.0" "c2 1.0" "c3 1.0 8" "c3 1.0 64" "c4 0.25" "c5 1.0 0 0"; do
  timeout 900 python scripts/run_config.py $args >> "$out" 2> gpurun_out/sweep_err.log || echo "{\"failed\": \"$args\"}" >> "$out"
done
