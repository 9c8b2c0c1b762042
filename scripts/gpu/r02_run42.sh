# round-2 (session 5): c5 with the contour's conjugate symmetry (shifts 0..3 solved, 4..7 their conjugates, checked on the host)
set -x
mkdir -p gpurun_out
timeout 1200 python scripts/run_c5_shifts.py 1.0 conj > gpurun_out/r42_c5_conj.jsonl 2> gpurun_out/r42_c5.err; echo "c5 rc=$?"
cut -c1-330 gpurun_out/r42_c5_conj.jsonl; tail -3 gpurun_out/r42_c5.err
