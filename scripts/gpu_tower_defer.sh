# deferred tower dW vs single-stream tower, W=1 DLRM default bench
export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for D in 1 0; do
NEST_TOWER_DEFER_DW=$D timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/td$D.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/td$D.log') if x.startswith('{')][-1]; d=json.loads(l)
st=d['stages']; print('defer=$D', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms e2e', round(d['e2e']['value']/1e6,2), {k: round(v['ms_per_step'],3) for k,v in st.items()}, 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
