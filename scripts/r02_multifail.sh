for i in 1 2 3; do
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -rf -s 2>&1 > gpurun_out/multi_run_$i.log; tail -2 gpurun_out/multi_run_$i.log
grep -E "^FAILED|FAIL\]|MGPU FAILED|mismatch|Error:|Timeout|timed out|Traceback" gpurun_out/multi_run_$i.log | head -20
done
