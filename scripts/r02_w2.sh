# 2-GPU session: NCCL All2All anchor, W=2 bench (E+T N=1 + N=2, E), route exchange over the window, traces
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 300 $T --master-port 29501 scripts/nccl_a2a_anchor.py > gpurun_out/w2_a2a_anchor.json 2>gpurun_out/w2_a2a_anchor.err; tail -1 gpurun_out/w2_a2a_anchor.json
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/fwp_decomp.py > gpurun_out/fwp_decomp.json 2>&1; tail -1 gpurun_out/fwp_decomp.json
A="--gpus 2 --no-cpu-baseline --steps 30"
timeout 600 $T --master-port 29502 bench.py $A > gpurun_out/w2_bench.json 2>gpurun_out/w2_bench.err
NEST_ROUTE_XCHG=window timeout 600 $T --master-port 29503 bench.py $A > gpurun_out/w2_bench_rw.json 2>gpurun_out/w2_bench_rw.err
timeout 600 $T --master-port 29504 bench.py $A --no-e2e --no-fwp-compare --variant e --trace gpurun_out/w2_trace_e.json > gpurun_out/w2_trace_e.log 2>&1
timeout 600 $T --master-port 29505 bench.py $A --no-e2e --no-fwp-compare --trace gpurun_out/w2_trace_et.json > gpurun_out/w2_trace_et.log 2>&1
timeout 600 $T --master-port 29506 bench.py $A --no-e2e --no-fwp-compare --micro-batches 2 --trace gpurun_out/w2_trace_et_n2.json > gpurun_out/w2_trace_et_n2.log 2>&1
timeout 600 $T --master-port 29507 bench.py $A --no-e2e --no-fwp-compare --micro-batches 2 --variant e > gpurun_out/w2_e_n2.log 2>&1
python scripts/bsum.py gpurun_out/w2_bench.json gpurun_out/w2_bench_rw.json gpurun_out/w2_trace_e.log gpurun_out/w2_trace_et.log gpurun_out/w2_trace_et_n2.log gpurun_out/w2_e_n2.log
for f in e et et_n2; do python scripts/timeline.py gpurun_out/w2_trace_$f.json 2 > gpurun_out/w2_timeline_$f.txt; done
