# W=4 stage timelines (E+T and E), current defaults
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
A="--gpus 4 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 10"
timeout 600 $T --master-port 29815 bench.py $A --trace gpurun_out/w4tr_et.json > gpurun_out/w4tr_et.log 2>/dev/null
timeout 600 $T --master-port 29816 bench.py $A --variant e --trace gpurun_out/w4tr_e.json > gpurun_out/w4tr_e.log 2>/dev/null
for f in et e; do python scripts/timeline.py gpurun_out/w4tr_$f.json 2 > gpurun_out/w4tr_tl_$f.txt; done
