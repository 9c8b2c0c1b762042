set -x
timeout 300 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/gpu/sanitize_case.py c1 2>&1 | tail -5; echo "rc=$?"
