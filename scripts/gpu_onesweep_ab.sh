# r01g: one-sweep radix (decoupled look-back) vs the classic per-pass sort: parity + W=1 A/B + launch list
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d.get('embedding_only') or {}
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e.get('ms_per_step',0),3), {k: round(v,3) for k,v in e['stage_ms_per_step'].items()})"; }
for rep in 1 2; do
NEST_RADIX=classic timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/os_old_$rep.log 2>&1; summ gpurun_out/os_old_$rep.log classic$rep
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/os_new_$rep.log 2>&1; summ gpurun_out/os_new_$rep.log onesweep$rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/os_launches_e.csv \
  python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/os_ncu_e.log 2>&1; echo rc=$?
