export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_local_ranks.py -x -q -k "2-fused-early" 2>&1 | tail -2
A="--no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
timeout 300 python bench.py $A --trace gpurun_out/trace_et.json > gpurun_out/trace_et.log 2>&1
timeout 300 python bench.py $A --variant e --trace gpurun_out/trace_e.json > gpurun_out/trace_e.log 2>&1
python scripts/timeline.py gpurun_out/trace_et.json 2 > gpurun_out/timeline_et.txt
python scripts/timeline.py gpurun_out/trace_e.json 2 > gpurun_out/timeline_e.txt
python scripts/bsum.py gpurun_out/trace_et.log gpurun_out/trace_e.log
