T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 10"
timeout 600 $T --master-port 29781 bench.py $A --trace gpurun_out/dwbtr_et_on.json > gpurun_out/dwbtr_et_on.log 2>/dev/null
NEST_DIRECT_WB=0 timeout 600 $T --master-port 29782 bench.py $A --trace gpurun_out/dwbtr_et_off.json > gpurun_out/dwbtr_et_off.log 2>/dev/null
timeout 600 $T --master-port 29783 bench.py $A --variant e --trace gpurun_out/dwbtr_e_on.json > gpurun_out/dwbtr_e_on.log 2>/dev/null
for f in et_on et_off e_on; do python scripts/timeline.py gpurun_out/dwbtr_$f.json 2 > gpurun_out/dwbtr_tl_$f.txt; done
python scripts/bsum.py gpurun_out/dwbtr_*.log
