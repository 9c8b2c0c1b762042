# round-2 (session 5): c3 full size over P = 8, 16, 32, 64 (BASELINE configs[2]: "P=8..64") with clocks
set -x
mkdir -p gpurun_out
rm -f gpurun_out/r36_c3_P.jsonl
for P in 8 16 32 64; do timeout 600 python scripts/run_config.py c3 1.0 $P >> gpurun_out/r36_c3_P.jsonl 2>> gpurun_out/r36_c3_P.err; done
python - <<'PY'
import json
for l in open('gpurun_out/r36_c3_P.jsonl'):
    d=json.loads(l)
    print({k:(round(d[k],4) if isinstance(d.get(k),float) else d.get(k)) for k in ('P','t_lu','t_spikes','t_solve','iterations','apply_ms','residual_final')})
PY
