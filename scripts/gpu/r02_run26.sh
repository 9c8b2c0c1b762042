# round-2 (session 5): symmetric schedule incl. complex symmetric (c5) -- all GPU tests, componentwise report,
# c5 shifts 1 and 2 (short solves) for the LU time, c2 bench (non-symmetric: unchanged path)
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r26_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/r26_gpu_tests.log
timeout 600 python scripts/gpu/cw_report.py > gpurun_out/r26_cw.jsonl 2> gpurun_out/r26_cw.err; echo "cw rc=$?"
cut -c1-700 gpurun_out/r26_cw.jsonl
timeout 900 python scripts/run_c5_shifts.py 1.0 1 2 > gpurun_out/r26_c5_shifts_1_2.jsonl 2> gpurun_out/r26_c5.err; echo "c5 rc=$?"
cut -c1-600 gpurun_out/r26_c5_shifts_1_2.jsonl
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r26_bench_c2.json 2> gpurun_out/r26_bench_c2.err; echo "c2 rc=$?"
cut -c1-900 gpurun_out/r26_bench_c2.json
