set -x
timeout 300 python scripts/dev/misuse_probe.py 2>&1 | tail -20
