CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dlrm or bit_exact or error" 2>&1 | tail -2
for N in 1 2 4; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches $N > gpurun_out/e1_n$N.log 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29900+N)) bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/e2_n$N.log 2>&1
done
CUDA_VISIBLE_DEVICES=0 NEST_TOWER_SM_RESERVE=0 timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches 1 > gpurun_out/e1_n1_r0.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/e[12]_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"] or {}; st=d["stages"]
        print(f.split('/')[-1], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a.get("physical_ms_per_step",0),3), "exp", round(a.get("exposed_ms_per_step",0),3), "| tower", round(st["tower"]["ms_per_step"],3), round(st["tower"]["tflops"],0), "TF/s pool", round(st["pool"]["ms_per_step"],3), "seg", round(st["segsum"]["ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
