# round-2 (session 5): ncu --set full of the fused one-RHS apply launch (four partial sums per chunk), c3 P=64
set -x
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_solve_lu1 -s 1 -c 1 -o gpurun_out/ncu/r69_c3_apply python scripts/ncu_target.py c3 1.0 nosolve 64 > gpurun_out/ncu/r69.log 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/ncu/r69_c3_apply.ncu-rep 2>&1 | head -24
