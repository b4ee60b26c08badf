# r01g, 2 GPUs: trained tower (NEXT-4) -- parity W=1, multi-rank (AllReduce pin), E+T bench W=1/W=2 trained vs fixed
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,200}|FAILED|passed|failed" | head -20
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rf -k "2-fused-early]" -s 2>&1 | grep -E "tower-train|FAILED|passed|failed"
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'tower', round(d['stages']['tower']['ms_per_step'],3), 'dw', round(d['stages']['tower_dw']['ms_per_step'],3))"; }
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-fwp-compare --tower-train > gpurun_out/tt_w1.log 2>&1; summ gpurun_out/tt_w1.log w1_trained
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 40 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/tf_w1.log 2>&1; summ gpurun_out/tf_w1.log w1_fixed
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
  bench.py --gpus 2 --steps 40 --no-cpu-baseline --no-e2e --no-fwp-compare --tower-train > gpurun_out/tt_w2.log 2>&1; summ gpurun_out/tt_w2.log w2_trained
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29912 \
  bench.py --gpus 2 --steps 40 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/tf_w2.log 2>&1; summ gpurun_out/tf_w2.log w2_fixed
