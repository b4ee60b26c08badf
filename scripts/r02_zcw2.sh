T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29791 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/zc_w2.json 2>gpurun_out/zc_w2.err; echo rc=$?
python scripts/bsum.py gpurun_out/zc_w2.json
NEST_ZERO_COPY=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "2-fused-early]" 2>&1 | tail -2
