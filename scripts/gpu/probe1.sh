set -x
nproc; free -g; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import os; print(len(os.sched_getaffinity(0)))"
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py 2>&1 | tail -15
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -k "full_c" 2>&1 | tail -8
timeout 300 python -m pytest tests/test_gpu_lu_int8.py -m gpu -q -s -k componentwise 2>&1 | tail -15
timeout 600 python scripts/run_config.py c3 1.0 64 > gpurun_out/p1_c3p64.json 2>gpurun_out/p1_c3p64.err; tail -c 3000 gpurun_out/p1_c3p64.json
