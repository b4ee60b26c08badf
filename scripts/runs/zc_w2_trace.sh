T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 10 --config dbp_stress --reuse 0.7"
NEST_ZERO_COPY=1 timeout 600 $T2 --master-port 29841 bench.py $A --trace gpurun_out/zcw2_et.json > gpurun_out/zcw2_et.log 2>gpurun_out/zcw2_et.err
python scripts/timeline.py gpurun_out/zcw2_et.json 2 > gpurun_out/zcw2_tl_et.txt
NEST_ZERO_COPY=1 timeout 600 $T2 --master-port 29842 bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --steps 10 --trace gpurun_out/zcw2d_et.json > gpurun_out/zcw2d_et.log 2>/dev/null
python scripts/timeline.py gpurun_out/zcw2d_et.json 2 > gpurun_out/zcw2d_tl_et.txt
python scripts/bsum.py gpurun_out/zcw2_et.log gpurun_out/zcw2d_et.log
