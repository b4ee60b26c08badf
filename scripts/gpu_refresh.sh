# r01g: compacting refresh kernel -- parity, default bench (driver-like), launch list (E)
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/rf2_bench.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/rf2_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
e=d['embedding_only']
print(round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value']/1e6,3), 'roof', round(d['roofline']['frac'],3), 'E', round(e['ms_per_step'],3), {k: round(v,3) for k,v in e['stage_ms_per_step'].items()})"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf2_launches_e.csv \
  python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/rf2_ncu_e.log 2>&1; echo rc=$?
