export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
timeout 300 python bench.py $A --variant e --trace gpurun_out/trace3_e.json > gpurun_out/trace3_e.log 2>&1
timeout 300 python bench.py $A --trace gpurun_out/trace3_et.json > gpurun_out/trace3_et.log 2>&1
python scripts/timeline.py gpurun_out/trace3_e.json 3 > gpurun_out/timeline3_e.txt
python scripts/timeline.py gpurun_out/trace3_et.json 3 > gpurun_out/timeline3_et.txt
python scripts/bsum.py gpurun_out/trace3_e.log gpurun_out/trace3_et.log
