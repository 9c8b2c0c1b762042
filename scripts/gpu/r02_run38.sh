# round-2 (session 5): upload with the copies overlapped with the host validation -- all GPU tests, c3 bench (e2e)
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r38_gpu_tests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/r38_gpu_tests.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r38_bench.json 2> gpurun_out/r38_bench.err; echo "bench rc=$?"
cut -c1-1300 gpurun_out/r38_bench.json
timeout 600 python scripts/run_config.py c3 1.0 64 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('t_upload','t_factorize_wall','t_factorize','t_lu','t_spikes','t_solve')})"
