# 4-GPU session: NCCL anchor, default bench at W=4 and W=2 on the same box, multi-GPU parity at W=4
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 300 $T4 --master-port 29501 scripts/nccl_a2a_anchor.py > gpurun_out/w4_a2a_anchor.json 2>/dev/null; tail -1 gpurun_out/w4_a2a_anchor.json
timeout 900 $T4 --master-port 29502 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/w4_bench.json 2>gpurun_out/w4_bench.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29503 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/w4box_w2_bench.json 2>/dev/null
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/w4box_w1_bench.json 2>/dev/null
python scripts/bsum.py gpurun_out/w4_bench.json gpurun_out/w4box_w2_bench.json gpurun_out/w4box_w1_bench.json
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -k "4-" 2>&1 | tail -3
