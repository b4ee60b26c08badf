export CUDA_VISIBLE_DEVICES=0
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep "Model name"; nproc
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r02_base_bench.json 2>gpurun_out/r02_base_bench.err; echo bench rc=$?
tail -c 300 gpurun_out/r02_base_bench.json
