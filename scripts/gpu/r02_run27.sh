# round-2 (session 5): where the symmetric c3 LU goes -- ncu launch list of one factorization, LU variants (sym on / off, pairs / quads)
set -x
mkdir -p gpurun_out/ncu
timeout 900 python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/r27_plain.log 2>&1; echo "plain rc=$?"
tail -2 gpurun_out/r27_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/ncu/r27_launches_fact.csv python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/ncu/r27_launch.log 2>&1; echo "launch rc=$?"
python scripts/ncu_summary.py gpurun_out/ncu/r27_launches_fact.csv > gpurun_out/r27_launches_fact.txt 2>&1 || true
head -30 gpurun_out/r27_launches_fact.txt
timeout 1500 python scripts/lu_variants.py c3 1.0 64 3 > gpurun_out/r27_lu_c3.jsonl 2>&1; echo "lu rc=$?"
cut -c1-260 gpurun_out/r27_lu_c3.jsonl
LRS_LU_SYM=0 timeout 600 python scripts/lu_variants.py c2 1.0 8 3 > gpurun_out/r27_lu_c2.jsonl 2>&1; echo "lu c2 rc=$?"
cut -c1-260 gpurun_out/r27_lu_c2.jsonl
