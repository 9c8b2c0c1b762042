# round-2 re-entry: GPU tests, smoke, bench (c3 P=64 + c2), reference arm, launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r1_gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r1_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r1_bench.json
timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r1_bench_c2.json 2> gpurun_out/r1_bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r1_bench_ref.json 2> gpurun_out/r1_bench_ref.err; echo "ref rc=$?"
