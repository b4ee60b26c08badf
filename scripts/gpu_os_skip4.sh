# r01g, 4 GPUs: one-sweep radix + gather-skip A/B at W=1/2/4, parity, multi-rank parity
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf 2>&1 | grep -E "^E  .{0,160}|FAILED|passed|failed" | head -20
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -rf -k "fused-early-2 or 4" 2>&1 | grep -E "FAILED|passed|failed"
summ() { python -c "
import json,sys; l=[x for x in open('$1') if x.startswith('{')][-1]; d=json.loads(l)
e=d.get('embedding_only') or {}
print('$2', round(d['value']/1e6,3), 'Msps', round(d['ms_per_step'],3), 'ms clk', d['clocks']['sm_mhz'], 'E', round(e.get('ms_per_step',0),3), 'sort', round(d['stages']['sort']['ms_per_step'],3), 'Esort', round(e['stage_ms_per_step']['sort'],3))"; }
for rep in 1 2; do
CUDA_VISIBLE_DEVICES=0 NEST_RADIX=classic timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/o4_w1c_$rep.log 2>&1; summ gpurun_out/o4_w1c_$rep.log w1_classic$rep
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/o4_w1_$rep.log 2>&1; summ gpurun_out/o4_w1_$rep.log w1_onesweep$rep
done
run() { W=$1; tag=$2; shift 2; env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) \
  bench.py --gpus $W --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/o4_$tag.log 2>&1; summ gpurun_out/o4_$tag.log $tag; }
run 4 w4_skip1 NEST_GATHER_SKIP=1
run 4 w4_skip0 NEST_GATHER_SKIP=0
run 4 w4_skip1_classic NEST_GATHER_SKIP=1 NEST_RADIX=classic
run 2 w2_skip1 NEST_GATHER_SKIP=1
run 2 w2_skip0 NEST_GATHER_SKIP=0
run 4 w4_skip0_b NEST_GATHER_SKIP=0
run 4 w4_skip1_b NEST_GATHER_SKIP=1
