# round-2 (session 5): ncu launch list of the bench command with the symmetric schedule
set -x
mkdir -p gpurun_out/ncu
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/ncu/r43_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu/r43_launch.log 2>&1; echo "launch rc=$?"
python scripts/ncu_summary.py gpurun_out/ncu/r43_launches_c3.csv > gpurun_out/r43_launches_c3.txt 2>&1
head -30 gpurun_out/r43_launches_c3.txt
