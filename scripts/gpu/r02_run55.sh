# round-2 (session 5): compact FP32 factor copy -- mixed-precision tests, then c3 P=64 at full size with factor_fp32
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 900 python scripts/run_mixed.py c3 1.0 64 > gpurun_out/r55_mixed_c3.jsonl 2> gpurun_out/r55_mixed.err; echo "mixed rc=$?"
cut -c1-700 gpurun_out/r55_mixed_c3.jsonl; tail -3 gpurun_out/r55_mixed.err
