# round-2: complex INT8 LU (realified pairs): INT8 tests incl. c5, complex / fullsize / pivoting suites, c5 shifts 0 and 3
set -x
timeout 1500 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_complex.py tests/test_gpu_fullsize.py tests/test_gpu_pivoting.py tests/test_gpu_coupling.py -q -p no:cacheprovider > gpurun_out/r13_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r13_tests.log | tail -12
timeout 900 python scripts/run_c5_shifts.py 1.0 0 3 > gpurun_out/r13_c5.jsonl 2> gpurun_out/r13_c5.err; echo "c5 rc=$?"
cut -c1-330 gpurun_out/r13_c5.jsonl; tail -3 gpurun_out/r13_c5.err
