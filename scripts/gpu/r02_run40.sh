set -x
timeout 600 python scripts/dev/e2e_probe2.py 2>&1 | tail -6
