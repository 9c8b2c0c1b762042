set -x
LRS_UPLOAD_TRACE=1 timeout 600 python scripts/dev/upload_probe.py c3 2>&1 | tail -14
