# r01g: streamed expand (unpooled) -- parity + gen-rec W=1 A/B
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()}, 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))"; }
for rep in 1 2; do
NEST_POOL=bag timeout 900 python bench.py --config genrec --steps 10 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/ex_old_$rep.log 2>&1; summ gpurun_out/ex_old_$rep.log expand_rows$rep
timeout 900 python bench.py --config genrec --steps 10 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/ex_new_$rep.log 2>&1; summ gpurun_out/ex_new_$rep.log expand_stream$rep
done
timeout 900 python bench.py --config genrec --steps 10 > gpurun_out/ex_full.log 2>&1; tail -c 400 gpurun_out/ex_full.log
