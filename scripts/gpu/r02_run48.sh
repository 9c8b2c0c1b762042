set -x
mkdir -p gpurun_out
timeout 600 python scripts/dev/setup_profile.py c4 0.25 2>&1 | tail -3 | cut -c1-900
timeout 600 python scripts/dev/setup_profile.py c3 1.0 64 2>&1 | tail -1 | cut -c1-900
