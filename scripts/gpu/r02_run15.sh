# round-2: 16-warp complex forward sweeps: complex suites, c5 shifts 0 and 3, ncu of the sweep
set -x
mkdir -p gpurun_out/ncu
timeout 1500 python -m pytest tests/test_gpu_complex.py tests/test_gpu_fullsize.py tests/test_gpu_pivoting.py tests/test_gpu_coupling.py tests/test_gpu_lu_int8.py -q -p no:cacheprovider > gpurun_out/r15_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r15_tests.log | tail -8
timeout 900 python scripts/run_c5_shifts.py 1.0 0 3 > gpurun_out/r15_c5.jsonl 2> gpurun_out/r15_c5.err; echo "c5 rc=$?"
cut -c1-330 gpurun_out/r15_c5.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_solve_z -s 8 -c 1 -o gpurun_out/ncu/r15_c5_zsolve python scripts/ncu_target.py c5 1.0 nosolve > gpurun_out/ncu/r15_zsolve.log 2>&1; echo "zsolve rc=$?"
