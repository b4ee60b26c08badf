export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "bench_path" --durations=3 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/r02_bench2.json 2>gpurun_out/r02_bench2.err; echo bench rc=$?
