# W=1 DLRM E+T: tower SM reserve x micro-batches (with deferred dW)
export CUDA_VISIBLE_DEVICES=0
for R in 0 16 24 40; do for N in 1 2; do
NEST_TOWER_SM_RESERVE=$R timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/ov_${R}_$N.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/ov_${R}_$N.log') if x.startswith('{')][-1]; d=json.loads(l)
st=d['stages']; print('reserve=$R N=$N', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_step'],3) for k,v in st.items() if k in ('pool','segsum','tower','tower_dw','route','sort')})"
done; done
