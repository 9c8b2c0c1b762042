set -x
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python scripts/spmv_ab.py 2>&1 | tail -3
# launch list of one bench step (c3 P=64), then ncu captures (one ncu tool per call)
timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/p6_bench_plain.json 2> gpurun_out/p6_bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/p6_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/p6_target.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:band_solve -s 4 -c 2 -o gpurun_out/r02_c3_apply python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/p6_ncu_apply.log 2>&1
echo "apply ncu rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lu_i8_gemm -s 30 -c 1 -o gpurun_out/r02_c3_lu_i8 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/p6_ncu_lu.log 2>&1
echo "lu ncu rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv -s 2 -c 1 -o gpurun_out/r02_c3_spmv python scripts/ncu_target.py c3 1.0 solve 64 > gpurun_out/p6_ncu_spmv.log 2>&1
echo "spmv ncu rc=$?"
