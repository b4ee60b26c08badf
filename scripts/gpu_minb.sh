# r01g: k_segsum_range at 3 vs 2 resident blocks (80 regs + small spills vs 98 regs), W=1 E and E+T, A/B/A/B
export CUDA_VISIBLE_DEVICES=0
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d['embedding_only']
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e['ms_per_step'],3), 'segsum', round(e['stage_ms_per_step']['segsum'],3), 'frac', round(d['roofline']['frac'],3), round(e['roofline']['frac'],3))"; }
for rep in 1 2; do
for v in 2 3; do
cp paper_2604_06956_b200/alt/libnest_minb$v.so paper_2604_06956_b200/libnest.so
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/mb_${v}_$rep.log 2>&1; summ gpurun_out/mb_${v}_$rep.log minb${v}_$rep
done
done
cp paper_2604_06956_b200/alt/libnest_minb3.so paper_2604_06956_b200/libnest.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "dlrm_full or giant or dyadic or adagrad" 2>&1 | tail -1
