# hot-final block size A/B, W=1 (E-only and E+T stage times)
export CUDA_VISIBLE_DEVICES=0
for rep in 1 2; do for H in 1024 256; do
NEST_HOT_THREADS=$H timeout 600 python bench.py --steps 60 --no-cpu-baseline --no-e2e > gpurun_out/h_$H.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/h_$H.log') if x.startswith('{')][-1]; d=json.loads(l)
print('rep=$rep hot=$H', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'segsum', round(d['stages']['segsum']['ms_per_step'],3), 'roof', round(d['roofline']['frac'],3), 'emb_only', round(d['embedding_only']['ms_per_step'],3), 'E segsum', round(d['embedding_only']['stage_ms_per_step']['segsum'],3))"
done; done
