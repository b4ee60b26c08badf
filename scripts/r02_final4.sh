timeout 2400 python -m pytest tests/test_gpu_multi.py -q -rs 2>&1 | tail -4
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
timeout 900 $T4 --master-port 29951 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/final_w4.json 2>/dev/null
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29952 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/final_w2.json 2>/dev/null
python scripts/bsum.py gpurun_out/final_w4.json gpurun_out/final_w2.json
