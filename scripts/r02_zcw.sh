export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests/test_gpu_local_ranks.py -q -x -k "zerocopy" 2>&1 | tail -2
NEST_ZERO_COPY=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "not route_w1_bit_exact" 2>&1 | tail -3
