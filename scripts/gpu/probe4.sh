set -x
timeout 600 python scripts/gpu/cw_report.py > gpurun_out/p4_cw.jsonl 2>&1; cat gpurun_out/p4_cw.jsonl | tail -3
timeout 1200 python bench.py --steps 2 --warmup 1 > gpurun_out/p4_bench.json 2> gpurun_out/p4_bench.err; tail -c 8000 gpurun_out/p4_bench.json; tail -5 gpurun_out/p4_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/p4_ref.json 2>&1; tail -c 3000 gpurun_out/p4_ref.json
