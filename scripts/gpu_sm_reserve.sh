# r01g: tower SM-count target (NEST_TOWER_SM_RESERVE) at W=1 E+T, A/B/C x2
export CUDA_VISIBLE_DEVICES=0
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'tower', round(d['stages']['tower']['ms_per_step'],3), round(d['stages']['tower_dw']['ms_per_step'],3), 'roof', round(d['roofline']['frac'],3))"; }
for rep in 1 2; do
for rs in 24 0 12; do
NEST_TOWER_SM_RESERVE=$rs timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/smr_${rs}_$rep.log 2>&1; summ gpurun_out/smr_${rs}_$rep.log reserve${rs}_$rep
done
done
