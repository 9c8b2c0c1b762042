set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k full_size_properties -x -q -s -p no:cacheprovider > gpurun_out/r41_props.log 2>&1; echo "rc=$?"
grep -E "round trip|linearity|passed|failed|Error|assert" gpurun_out/r41_props.log | head -30
