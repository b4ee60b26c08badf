# compute-sanitizer on the tiny pipelined path: W=1 N=2 (smoke) and W=2 ranks
# on one GPU (fused transport, every exchange over the peer windows)
export CUDA_VISIBLE_DEVICES=0
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/san_w1_$tool.log 2>&1
  echo "w1 $tool rc=$?"; tail -3 gpurun_out/san_w1_$tool.log
done
for tool in memcheck synccheck; do
  NEST_MGPU_SAME_DEVICE=1 NEST_MGPU_BIG=0 NEST_MGPU_ONLY=tiny-P1-N2 timeout 1200 $CS --tool $tool --target-processes all \
    --error-exitcode 9 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 \
    --master-port 29611 tests/mgpu_worker.py > gpurun_out/san_w2_$tool.log 2>&1
  echo "w2 $tool rc=$?"; grep -E "ERROR SUMMARY|OK|FAIL" gpurun_out/san_w2_$tool.log | head -8
done
