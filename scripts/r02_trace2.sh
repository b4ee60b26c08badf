export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
NEST_TOWER_DW_AFTER_BWD=1 timeout 300 python bench.py $A --trace gpurun_out/trace_et_dwa.json > gpurun_out/trace_et_dwa.log 2>&1
python scripts/timeline.py gpurun_out/trace_et_dwa.json 2 > gpurun_out/timeline_et_dwa.txt
python scripts/bsum.py gpurun_out/trace_et_dwa.log
