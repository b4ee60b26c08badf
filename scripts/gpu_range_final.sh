# r01g: streaming pool + range segment-sum as defaults: parity, A/B vs r01 kernels, launch list, ncu --set full
export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "FAILED|passed|failed" | head -20
NEST_SEGSUM=range python scripts/ada_debug.py 1 1 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d['embedding_only']
print('$2', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e['ms_per_step'],3), {k: round(v,3) for k,v in e['stage_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],3), round(e['roofline']['frac'],3))"; }
for rep in 1 2 3; do
NEST_POOL=bag NEST_SEGSUM=chunks timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/rf_old_$rep.log 2>&1; summ gpurun_out/rf_old_$rep.log old$rep
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/rf_new_$rep.log 2>&1; summ gpurun_out/rf_new_$rep.log new$rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_e.csv \
  python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/rf_ncu_e.log 2>&1
echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_et.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/rf_ncu_et.log 2>&1
echo ncu et rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_seg|k_pool|k_gather|k_refresh" -s 10 -c 10 \
  -o gpurun_out/rf_full -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/rf_ncu_full.log 2>&1
echo ncu full rc=$?
