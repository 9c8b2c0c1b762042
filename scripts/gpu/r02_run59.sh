# round-2 (session 5): bench.py --config c5 (one contour shift per rank; shift 1 here via --steps 1) still runs with the symmetric schedule
set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r59_bench_c5.json 2> gpurun_out/r59_bench_c5.err; echo "rc=$?"
cut -c1-1200 gpurun_out/r59_bench_c5.json; tail -3 gpurun_out/r59_bench_c5.err
