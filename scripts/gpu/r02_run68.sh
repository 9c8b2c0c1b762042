# round-2 (session 5): is the FP64 one-RHS sweep bound by its single FMA chain? NA partial sums per chunk (build/var_accN) vs one
set -x
for rep in 1 2; do
for lib in "" build/var_acc2/liblrspike_cuda.so build/var_acc4/liblrspike_cuda.so build/var_acc8/liblrspike_cuda.so; do
LRS_LIB=$lib timeout 300 python scripts/run_config.py c3 1.0 64 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('lib', '$lib' or 'default', 'apply_ms', round(d['apply_ms'],3), 't_solve', round(d['t_solve'],3), 'it', d['iterations'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
for lib in "" build/var_acc4/liblrspike_cuda.so; do
LRS_LIB=$lib timeout 300 python scripts/run_config.py c2 1.0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2 lib', '$lib' or 'default', 'apply_ms', round(d['apply_ms'],3), 't_solve', round(d['t_solve'],4), 'it', d['iterations'])"
done
