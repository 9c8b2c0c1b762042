# round-2 (session 5): final-build refresh of c3 over P = 8..64 and the mixed-precision c3 run
set -x
mkdir -p gpurun_out
rm -f gpurun_out/r70_c3_P.jsonl
for P in 8 16 32 64; do timeout 600 python scripts/run_config.py c3 1.0 $P >> gpurun_out/r70_c3_P.jsonl 2>/dev/null; done
python - <<'PY'
import json
for l in open('gpurun_out/r70_c3_P.jsonl'):
    d=json.loads(l)
    print({k:(round(d[k],4) if isinstance(d.get(k),float) else d.get(k)) for k in ('P','t_lu','t_spikes','t_solve','iterations','apply_ms')})
PY
timeout 900 python scripts/run_mixed.py c3 1.0 64 > gpurun_out/r70_mixed_c3.jsonl 2>/dev/null; cut -c1-330 gpurun_out/r70_mixed_c3.jsonl
