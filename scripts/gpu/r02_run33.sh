# round-2 (session 5): SM clocks / power during the LU (the LU runs ~20% slower on today's boxes than in session 4)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,power.limit,power.max_limit,power.default_limit,clocks.max.sm,clocks.max.mem,vbios_version,driver_version --format=csv
(nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/r33_smi.csv) &
SMI=$!
LRS_VARIANT_CHILD=1 timeout 600 python scripts/lu_variants.py c3 1.0 64 6 > gpurun_out/r33_lu_c3.json 2>&1
LRS_VARIANT_CHILD=1 LRS_LU_SYM=0 timeout 600 python scripts/lu_variants.py c3 1.0 64 4 > gpurun_out/r33_lu_c3_nosym.json 2>&1
kill $SMI
cut -c1-300 gpurun_out/r33_lu_c3.json; cut -c1-300 gpurun_out/r33_lu_c3_nosym.json
sort gpurun_out/r33_smi.csv | uniq -c | sort -rn | head -25
