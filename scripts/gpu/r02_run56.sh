# round-2 (session 5): FP32 one-RHS sweep with four partial sums per chunk -- mixed tests, parity / fullsize / determinism, c3 mixed
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_fused_sweeps.py tests/test_gpu_variants.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 900 python scripts/run_mixed.py c3 1.0 64 > gpurun_out/r56_mixed_c3.jsonl 2> gpurun_out/r56_mixed.err; echo "mixed rc=$?"
cut -c1-420 gpurun_out/r56_mixed_c3.jsonl
