set -x
for rep in 1 2 3; do for t in 8 2; do
LRS_I8_TPC3=$t timeout 300 python bench.py --config c2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('TPC3', $t, round(d['value'],4), round(d['t_lu_s'],4), round(d['e2e']['value'],4))"
done; done
