# owner update over the listed multi-contributor keys (new) vs a skip test over every owner key (libnest_skip.so)
timeout 1500 python -m pytest tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "fused-early or fused-window or no-nccl" 2>&1 | tail -2
GPUS=2 bash scripts/runs/ab.sh 2 dl "list" "skip NEST_LIB=paper_2604_06956_b200/libnest_skip.so" -- --no-e2e --steps 30 --no-fwp-compare --variant e
GPUS=2 bash scripts/runs/ab.sh 2 dlet "list" "skip NEST_LIB=paper_2604_06956_b200/libnest_skip.so" -- --no-e2e --steps 50 --no-fwp-compare
for f in gpurun_out/dl_*.json gpurun_out/dlet_*.json; do python -c "
import json,sys
f=sys.argv[1]
d=json.loads([l for l in open(f).read().splitlines() if l.startswith('{')][-1]); st=d['stages']
print(f.split('/')[-1], 'ms/step', round(d['ms_per_step'],3), 'update', round(st['update']['ms_per_step'],3))
" $f; done
