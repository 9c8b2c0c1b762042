# round-2: quad look-ahead in pair form; slice kernel; LU variants; factorization launch list
set -x
mkdir -p gpurun_out/ncu
timeout 1200 python -m pytest tests/test_gpu_lu_int8.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/r10_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r10_tests.log | tail -10
timeout 1200 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r10_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-200 gpurun_out/r10_lu_c3.jsonl
timeout 600 python scripts/lu_variants.py c2 1.0 8 3 > gpurun_out/r10_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-200 gpurun_out/r10_lu_c2.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/ncu/r10_launches_fact.csv python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/ncu/r10_launch.log 2>&1; echo "launch rc=$?"
python scripts/ncu_summary.py gpurun_out/ncu/r10_launches_fact.csv | head -30
