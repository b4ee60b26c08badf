export NEST_LANES=2
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "train_w1_dyadic or realistic or clustered" 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29960 tests/mgpu_worker.py > gpurun_out/mgpu_l2.log 2>&1; echo mgpu_rc=$?; grep -E "ALL OK|FAIL|mismatch" gpurun_out/mgpu_l2.log | head -3
i=0
for M in fused ce; do for N in 2 4; do for R in 0 24; do
i=$((i+1))
NEST_A2A=$M NEST_TOWER_SM_RESERVE=$R timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29900+i)) bench.py --gpus 4 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/l2_${M}_n${N}_r$R.log 2>&1; echo $M N=$N R=$R rc=$?
done; done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/l2_*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"]; st=d["stages"]
        print(f.split('/')[-1][3:-4], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "| tower", round(st["tower"]["ms_per_step"],3), "pool", round(st["pool"]["ms_per_step"],3), "emb", round(st["emb_a2a"]["ms_per_step"],3), "grad", round(st["grad_a2a"]["ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
