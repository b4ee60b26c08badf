# r01g: bulk-copy (TMA) pool / segment-sum: GPU parity (all forms), A/B vs staged and the r01 kernels, ncu
export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,200}|FAILED|passed|failed" | head -30
for form in stage range; do
NEST_SEGSUM=$form NEST_POOL=$( [ $form = range ] && echo stream || echo stage ) timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "giant or dlrm_full or dims or hot_segments or adagrad or dyadic" 2>&1 | grep -E "FAILED|passed|failed" | sed "s/^/[$form] /" | head
done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d['embedding_only']
print('$2', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e['ms_per_step'],3), {k: round(v,3) for k,v in e['stage_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3), round(e['roofline']['frac'],3))"; }
for rep in 1 2; do
NEST_POOL=bag NEST_SEGSUM=chunks timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bab_old_$rep.log 2>&1; summ gpurun_out/bab_old_$rep.log old$rep
NEST_POOL=stage NEST_SEGSUM=stage timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bab_stage_$rep.log 2>&1; summ gpurun_out/bab_stage_$rep.log stage$rep
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bab_bulk_$rep.log 2>&1; summ gpurun_out/bab_bulk_$rep.log bulk$rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bab_launches_e.csv \
  python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/bab_ncu_e.log 2>&1
echo ncu rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_segsum_bulk|k_pool_bulk|k_segsum_fix" -s 6 -c 4 \
  -o gpurun_out/bab_full -f python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/bab_ncu_full.log 2>&1
echo ncu full rc=$?
