# the whole -m gpu suite on a 4-GPU box (multi-GPU parity at W = 2 and 4 included)
timeout 2700 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 | tee gpurun_out/gpu_tests_4gpu.log
