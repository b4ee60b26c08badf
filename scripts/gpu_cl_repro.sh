# clustered Zipf-0.8 N=4 at W=2 (was an illegal access) + clustering parity
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster" 2>&1 | tail -1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29711 \
  bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-fwp-compare --zipf 0.8 --micro-batches 4 --schedule clustered > gpurun_out/rp_1.log 2>&1
echo "rc=$?"; grep -h -m2 "NestError\|illegal" gpurun_out/rp_1.log | cut -c1-200
python -c "
import json; l=[x for x in open('gpurun_out/rp_1.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; schedule', round(d['stages']['schedule']['ms_per_step'],3), 'alpha', round(d['fwp']['alpha'],3))"
