export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --no-fwp-compare --steps 10"
timeout 300 python bench.py $A --trace gpurun_out/trace_et.json > gpurun_out/trace_et.log 2>&1
timeout 300 python bench.py $A --variant e --trace gpurun_out/trace_e.json > gpurun_out/trace_e.log 2>&1
python scripts/timeline.py gpurun_out/trace_et.json 2 > gpurun_out/timeline_et.txt
python scripts/timeline.py gpurun_out/trace_e.json 2 > gpurun_out/timeline_e.txt
python scripts/bsum.py gpurun_out/trace_et.log gpurun_out/trace_e.log
