# compute-sanitizer tiers on small cases (profiles/r02_sanitizer.txt)
mkdir -p gpurun_out/san
for case in c1 c2 c5; do
  for tool in memcheck racecheck synccheck initcheck; do
    echo "== $tool $case"
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python scripts/gpu/sanitize_case.py $case > gpurun_out/san/${tool}_${case}.log 2>&1
    echo "rc=$?"; tail -4 gpurun_out/san/${tool}_${case}.log
  done
done
