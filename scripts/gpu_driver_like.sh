# what the driver runs at round end (1 GPU), plus the 2-GPU pytest
CUDA_VISIBLE_DEVICES=0 timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -c 600 gpurun_out/bench_default.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?; tail -c 400 gpurun_out/bench_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29977 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_default_w2.log 2>&1; echo bench_w2_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29978 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ref_w2.log 2>&1; echo ref_w2_rc=$?; grep -c impl gpurun_out/bench_ref_w2.log
