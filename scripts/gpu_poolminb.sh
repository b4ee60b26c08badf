# r01g: k_pool_stream resident blocks 4 (62 regs) / 5 (<=51) / 6 (40 + spills), W=1 E and E+T, x2
export CUDA_VISIBLE_DEVICES=0
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d['embedding_only']
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e['ms_per_step'],3), 'pool', round(d['stages']['pool']['ms_per_step'],3), round(e['stage_ms_per_step']['pool'],3))"; }
for rep in 1 2; do
for v in 4 5 6; do
cp paper_2604_06956_b200/alt/libnest_pool$v.so paper_2604_06956_b200/libnest.so
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/pm_${v}_$rep.log 2>&1; summ gpurun_out/pm_${v}_$rep.log pool_minb${v}_$rep
done
done
