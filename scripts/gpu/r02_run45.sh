set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pivoting.py -x -q -p no:cacheprovider > gpurun_out/r45_piv.log 2>&1; echo "rc=$?"
tail -25 gpurun_out/r45_piv.log
