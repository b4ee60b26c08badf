# alternating A/B of NEST_EARLY_PUSH at W=2 (100 timed steps each, 2 rounds)
for rep in 1 2; do for E in sm 0 ce; do
NEST_EARLY_PUSH=$E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --steps 100 --no-cpu-baseline --no-e2e --no-fwp-compare > gpurun_out/ab_$E.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/ab_$E.log') if x.startswith('{')][-1]; d=json.loads(l)
print('rep=$rep early=$E', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms', 'clk', d['clocks']['sm_mhz'])"
done; done
