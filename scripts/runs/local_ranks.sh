export CUDA_VISIBLE_DEVICES=0
run() { # tag world, extra env...
  tag=$1; w=$2; shift; shift
  env NEST_MGPU_SAME_DEVICE=1 NEST_MGPU_DUMP_AFTER=200 "$@" timeout 250 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$w \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) tests/mgpu_worker.py > gpurun_out/loc_$tag.log 2>&1
  echo "== $tag rc=$?"; grep -E "OK|FAIL|mismatch|Error|error|Traceback|File \"/root|line [0-9]+, in" gpurun_out/loc_$tag.log | grep -v "elastic\|torch/distributed" | head -30
}
run w2big 2 NEST_MGPU_BIG=1
run w4small 4 NEST_MGPU_BIG=0
run w8small 8 NEST_MGPU_BIG=0
