T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --steps 30"
p=29620
for r in 1 2; do for ps in 0 1; do
  p=$((p+1))
  NEST_PUSH_STREAM=$ps timeout 600 $T --master-port $p bench.py $A > gpurun_out/push${ps}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/push*_r*.json
NEST_PUSH_STREAM=1 NEST_MGPU_BIG=0 timeout 900 $T --master-port 29640 tests/mgpu_worker.py 2>&1 | grep -E "OK|FAIL" | tail -8
