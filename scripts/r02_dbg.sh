T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
timeout 600 $T --master-port 29801 bench.py $A --zipf 0.8 > gpurun_out/dbg_z08.log 2>&1; echo rc=$?
grep -E "Error|error|NEST_ERR|Traceback" gpurun_out/dbg_z08.log | head -10
timeout 600 $T --master-port 29802 bench.py $A --micro-batches 4 > gpurun_out/dbg_n4.log 2>&1; echo rc=$?
grep -E "Error|error|NEST_ERR|Traceback" gpurun_out/dbg_n4.log | head -10
