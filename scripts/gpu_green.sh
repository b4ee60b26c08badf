# green-context lanes: functional check (tiny parity via smoke-like run) + W=2/W=4 perf
export NEST_TOWER_SM_RESERVE=0
CUDA_VISIBLE_DEVICES=0 NEST_GREEN_SMS=24 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "train_w1_dyadic" 2>&1 | tail -3
for G in 16 24 32; do for N in 2 4; do
NEST_GREEN_SMS=$G timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29870+G+N)) bench.py --gpus 4 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/g4_g${G}_n$N.log 2>&1; echo G=$G N=$N rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/g4_*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"]; st=d["stages"]
        print(f.split('/')[-1][3:-4], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "| tower", round(st["tower"]["ms_per_step"],3), "pool", round(st["pool"]["ms_per_step"],3), "emb", round(st["emb_a2a"]["ms_per_step"],3), "grad", round(st["grad_a2a"]["ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
tail -5 gpurun_out/g4_g24_n2.log
