T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 10 --variant e"
NEST_ROUTE_XCHG=window timeout 600 $T --master-port 29791 bench.py $A --trace gpurun_out/kxtr_e_win.json > gpurun_out/kxtr_e_win.log 2>/dev/null
python scripts/timeline.py gpurun_out/kxtr_e_win.json 2 > gpurun_out/kxtr_tl_e_win.txt
