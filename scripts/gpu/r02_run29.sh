# round-2 (session 5): evidence batch for the symmetric schedule -- c5 all eight shifts, ncu --set full of the
# symmetric INT8 bulk update (quad launch K=20) and the mirror kernel on c3 P=64, reference arm, config sweep
set -x
mkdir -p gpurun_out/ncu
FULL="ncu --set full --clock-control none --import-source on"
NT="python scripts/ncu_target.py"
timeout 1200 python scripts/run_c5_shifts.py 1.0 > gpurun_out/r29_c5_all_shifts.jsonl 2> gpurun_out/r29_c5.err; echo "c5 rc=$?"
tail -1 gpurun_out/r29_c5_all_shifts.jsonl | cut -c1-400
timeout 900 $FULL -k regex:lu_i8_gemm_kernel -s 16 -c 1 -o gpurun_out/ncu/r29_c3_lu_i8_sym $NT c3 1.0 nosolve 64 > gpurun_out/ncu/r29_i8.log 2>&1; echo "i8 rc=$?"
timeout 900 $FULL -k regex:lu_mirror_kernel -s 20 -c 1 -o gpurun_out/ncu/r29_c3_mirror $NT c3 1.0 nosolve 64 > gpurun_out/ncu/r29_mirror.log 2>&1; echo "mirror rc=$?"
for f in r29_c3_lu_i8_sym r29_c3_mirror; do python scripts/ncu_summary.py gpurun_out/ncu/$f.ncu-rep > gpurun_out/ncu/$f.txt 2>&1; done
head -30 gpurun_out/ncu/r29_c3_lu_i8_sym.txt
for c in "c1 1.0" "c2 1.0" "c3 1.0 8" "c4 0.25"; do timeout 600 python scripts/run_config.py $c >> gpurun_out/r29_configs.jsonl 2>> gpurun_out/r29_configs.err; done
cut -c1-500 gpurun_out/r29_configs.jsonl
timeout 1500 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r29_bench_reference.json 2> gpurun_out/r29_bench_reference.err; echo "ref rc=$?"
cut -c1-600 gpurun_out/r29_bench_reference.json
