# W>1 parity with the DBP-stress overlap case (local ranks on one GPU and over 2 GPUs)
timeout 1500 python -m pytest tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "fused-early or no-nccl" 2>&1 | tail -2
grep -h "dbp-overlap" gpurun_out/*.log 2>/dev/null | head -3
