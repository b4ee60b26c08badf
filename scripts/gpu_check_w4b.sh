for N in 1 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29840+N)) bench.py --gpus 4 --steps 30 --warmup 3 --no-e2e --micro-batches $N > gpurun_out/w4f_n$N.log 2>&1; echo N=$N rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/w4f_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"]; st=d["stages"]
        print(f.split('/')[-1], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "GB/s", round(a["nvlink_gbs_per_gpu"] or 0,1), "| nofwp", a["without_fwp"], "| tower", round(st["tower"]["ms_per_step"],3), "emb", round(st["emb_a2a"]["ms_per_step"],3), "grad", round(st["grad_a2a"]["ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
