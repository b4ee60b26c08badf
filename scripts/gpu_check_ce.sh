timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 tests/mgpu_worker.py > gpurun_out/mgpu_ce.log 2>&1; echo mgpu_ce_rc=$?
grep -E "OK|FAIL|mismatch|Error" gpurun_out/mgpu_ce.log | head
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; echo pytest_rc=$?; tail -15 gpurun_out/pytest_gpu.log
for N in 4 1; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29620+N)) bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/bench_ce_w2_n$N.log 2>&1; echo bench N=$N rc=$?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_ce_w2_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l)
        a=d["a2a"]; print(f, round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms a2a_phys", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "GB/s", round(a["nvlink_gbs_per_gpu"],1), "tower", round(d["stages"].get("tower",{}).get("ms_per_step",0),3))
    except Exception as e: print(f, "err", e)
PY
