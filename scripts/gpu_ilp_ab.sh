# A/B of NEST_ROW_ILP (pool / segment-sum interleave) on the W=1 DLRM bench
export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for V in e et; do for I in 1 2 4; do
NEST_ROW_ILP=$I timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --variant $V > gpurun_out/ilp_${V}_$I.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/ilp_${V}_$I.log') if x.startswith('{')][-1]; d=json.loads(l)
st=d['stages']; print('$V ilp=$I', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_step'],3) for k,v in st.items() if k in ('pool','segsum','gather','refresh','tower')}, 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done; done
