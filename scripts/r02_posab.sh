T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do timeout 600 $T --master-port $((29800+r)) bench.py $A > gpurun_out/pos_w2_r$r.json 2>/dev/null; done
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/pos_w1.json 2>/dev/null
python scripts/bsum.py gpurun_out/pos_w2_r*.json gpurun_out/pos_w1.json
NEST_MGPU_BIG=0 timeout 900 $T --master-port 29840 tests/mgpu_worker.py 2>&1 | grep -E "OK|FAIL" | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -2
