export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf "$@" 2>&1 | tail -60 > gpurun_out/parity_full.log
tail -60 gpurun_out/parity_full.log | grep -E "Error|assert|FAILED|passed|failed|^E " | head -60
