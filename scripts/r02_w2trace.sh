T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
timeout 600 $T --master-port 29511 bench.py $A --variant e --trace gpurun_out/w2b_trace_e.json > gpurun_out/w2b_trace_e.log 2>&1
timeout 600 $T --master-port 29512 bench.py $A --trace gpurun_out/w2b_trace_et.json > gpurun_out/w2b_trace_et.log 2>&1
python scripts/bsum.py gpurun_out/w2b_trace_e.log gpurun_out/w2b_trace_et.log
for f in e et; do python scripts/timeline.py gpurun_out/w2b_trace_$f.json 2 > gpurun_out/w2b_timeline_$f.txt; done
