export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster or edge" 2>&1 | tail -3
for N in 2 4 8; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --variant e --micro-batches $N --schedule clustered > gpurun_out/cl_n$N.log 2>&1
python -c "
import json; l=[x for x in open('gpurun_out/cl_n$N.log') if x.startswith('{')][-1]; d=json.loads(l)
print('N=$N', round(d['value']/1e6,2), 'Msps', round(d['ms_per_step'],3), 'ms; schedule', round(d['stages']['schedule']['ms_per_step'],3), 'ms; alpha', round(d['fwp']['alpha'],3))"
done
