# r01g: parity + gen-rec / DBP-stress W=1 with the current kernels (sort passes from U_s)
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()}, 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3))"; }
timeout 900 python bench.py --config genrec --steps 10 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/gr_range.log 2>&1; summ gpurun_out/gr_range.log genrec_range
NEST_SEGSUM=chunks timeout 900 python bench.py --config genrec --steps 10 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/gr_chunks.log 2>&1; summ gpurun_out/gr_chunks.log genrec_chunks
timeout 900 python bench.py --config dbp_stress --reuse 0.45 --steps 20 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/dbps.log 2>&1; summ gpurun_out/dbps.log dbp_stress_045
