# single-GPU parity (new refresh/update/runner), W=2 parity, then W=1 and W=2 bench sweeps
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5; echo pytest_rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29711 tests/mgpu_worker.py > gpurun_out/mgpu.log 2>&1; echo mgpu_rc=$?; grep -E "ALL OK|FAIL|mismatch" gpurun_out/mgpu.log | head -5
for R in 0 24 40; do for N in 1 4; do
  CUDA_VISIBLE_DEVICES=0 NEST_TOWER_SM_RESERVE=$R timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches $N > gpurun_out/b1_r${R}_n$N.log 2>&1
  NEST_TOWER_SM_RESERVE=$R timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29720+R+N)) bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/b2_r${R}_n$N.log 2>&1
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/b[12]_r*_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l)
        a=d["a2a"] or {}; st=d["stages"]
        print(f.split('/')[-1], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a.get("physical_ms_per_step",0),3), "exp", round(a.get("exposed_ms_per_step",0),3), "| tower", round(st.get("tower",{}).get("ms_per_step",0),3), "pool", round(st["pool"]["ms_per_step"],3), "seg", round(st["segsum"]["ms_per_step"],3), "upd", round(st["update"]["ms_per_step"],3), "busy", round(d["trace"]["compute_busy_ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
