# route exchange over the windows by default: multi-GPU parity (W=2 all transports, W=4) + W=2/4 E+T lines
timeout 2000 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 900 $T4 --master-port 29802 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/rw_w4_bench.json 2>gpurun_out/rw_w4_bench.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29803 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/rw_w2_bench.json 2>/dev/null
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/rw_w1_bench.json 2>/dev/null
python scripts/bsum.py gpurun_out/rw_w4_bench.json gpurun_out/rw_w2_bench.json gpurun_out/rw_w1_bench.json
