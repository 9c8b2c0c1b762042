# round-2: acceptance 8 / 10 on the GPU; the paper's single-precision preconditioner on c3
set -x
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_mixed.py -q -p no:cacheprovider > gpurun_out/r17_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r17_tests.log | tail -12
timeout 1200 python scripts/run_mixed.py c3 1.0 64 tests/golden/c3_s1_P64.npz > gpurun_out/r17_mixed_c3.jsonl 2> gpurun_out/r17_mixed_c3.err; echo "mixed rc=$?"
cat gpurun_out/r17_mixed_c3.jsonl; tail -3 gpurun_out/r17_mixed_c3.err
