set -x
timeout 300 python scripts/gpu/cw_debug.py 2>&1 | tail -20
mkdir -p gpurun_out/fx
LRS_FIXTURE_DIR=gpurun_out/fx LRS_ORACLE_THREADS=16 OPENBLAS_NUM_THREADS=1 timeout 2400 python tests/golden/make_full_fixtures.py c3:1.0:64 2>&1 | tail -5
free -g
