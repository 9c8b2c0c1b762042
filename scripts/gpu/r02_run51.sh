# round-2 (session 5): race detection by repetition at full size (c3 P=64 x 30, c2 x 40, c5 shift 0 x 8)
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/gpu/soak.py c3 1.0 64 30 > gpurun_out/r51_soak.jsonl 2> gpurun_out/r51_soak.err; echo "c3 rc=$?"
timeout 900 python scripts/gpu/soak.py c2 1.0 8 40 >> gpurun_out/r51_soak.jsonl 2>> gpurun_out/r51_soak.err; echo "c2 rc=$?"
timeout 1500 python scripts/gpu/soak.py c5 1.0 16 8 >> gpurun_out/r51_soak.jsonl 2>> gpurun_out/r51_soak.err; echo "c5 rc=$?"
cat gpurun_out/r51_soak.jsonl; tail -3 gpurun_out/r51_soak.err
