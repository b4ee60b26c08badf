timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 tests/mgpu_worker.py > gpurun_out/mgpu_fused.log 2>&1; echo mgpu_fused_rc=$?
grep -E "OK|FAIL|mismatch|Error" gpurun_out/mgpu_fused.log | head -8
for M in fused ce; do for N in 1 2; do
NEST_A2A=$M timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29630+N)) bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/f_${M}_n$N.log 2>&1; echo $M N=$N rc=$?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/f_*_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"]; st=d["stages"]
        print(f.split('/')[-1], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "GB/s", round(a["nvlink_gbs_per_gpu"] or 0,1), "| tower", round(st["tower"]["ms_per_step"],3), "| emb", round(st["emb_a2a"]["ms_per_step"],3), "grad", round(st["grad_a2a"]["ms_per_step"],3), "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"],3))
    except Exception as e: print(f, "err", e)
PY
