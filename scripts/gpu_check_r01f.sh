export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -3
timeout 300 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/h1.log 2>&1; echo bench_rc=$?
timeout 300 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --variant e > gpurun_out/h1e.log 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/h1.log","gpurun_out/h1e.log"]:
    l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); st=d["stages"]
    print(f, round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms |", " ".join(f"{k}={v['ms_per_step']:.3f}/{(v.get('frac_of_measured_hbm') or 0):.2f}" for k,v in st.items()), "| roof", d["roofline"]["kernel"], round(d["roofline"]["frac"],3))
PY
CMD="python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_h.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_pool|k_segsum_cold|k_reduce|k_gather" -s 12 -c 4 -o gpurun_out/prof_h $CMD > gpurun_out/ncu_h.log 2>&1; echo ncu=$?
