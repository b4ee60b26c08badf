# r01g: fresh-box check of the restored tree: GPU tests, smoke, default bench, E-only N=1 launch list
export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/g_bench.log 2>&1; tail -c 300 gpurun_out/g_bench.log
python -c "
import json; l=[x for x in open('gpurun_out/g_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks'], 'emb_only', round(d['embedding_only']['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['stages'].items()}, d['roofline']['frac'], d['embedding_only']['roofline']['frac'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_e.csv \
  python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare > gpurun_out/g_ncu_e.log 2>&1
echo ncu rc=$?
