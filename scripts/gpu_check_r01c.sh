CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5; echo pytest_rc=$?
for N in 1 4; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches $N > gpurun_out/c1_n$N.log 2>&1
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches $N --variant e > gpurun_out/c1e_n$N.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/c1*_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l)
        st=d["stages"]
        print(f.split('/')[-1], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms |", " ".join(f"{k}={v['ms_per_step']:.3f}/{(v.get('frac_of_measured_hbm') or 0):.2f}" for k,v in st.items()))
    except Exception as e: print(f, "err", e)
PY
