# end-of-round W = 4 / 2 / 1 default bench lines back to back on one 4-GPU box
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 900 $T4 --master-port 29871 bench.py --gpus 4 > gpurun_out/sf_w4_bench.json 2>gpurun_out/sf_w4_bench.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $T2 --master-port 29872 bench.py --gpus 2 > gpurun_out/sf_w2_bench.json 2>/dev/null
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/sf_w1_bench.json 2>/dev/null
python scripts/bsum.py gpurun_out/sf_w4_bench.json gpurun_out/sf_w2_bench.json gpurun_out/sf_w1_bench.json
