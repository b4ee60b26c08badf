# early push without the pending update's (stale) rows (new) vs pushing them too (libnest_prevpush.so)
timeout 1500 python -m pytest tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "fused-early or no-nccl" 2>&1 | tail -2
GPUS=2 bash scripts/runs/ab.sh 2 ps "skip" "all NEST_LIB=paper_2604_06956_b200/libnest_prevpush.so" -- --no-e2e --steps 30 --no-fwp-compare --variant e
GPUS=2 bash scripts/runs/ab.sh 2 pset "skip" "all NEST_LIB=paper_2604_06956_b200/libnest_prevpush.so" -- --no-e2e --steps 50 --no-fwp-compare
for f in gpurun_out/ps_*.json gpurun_out/pset_*.json; do python -c "
import json,sys
f=sys.argv[1]
d=json.loads([l for l in open(f).read().splitlines() if l.startswith('{')][-1]); st=d['stages']; a=d['a2a']
print(f.split('/')[-1], 'ms/step', round(d['ms_per_step'],3), 'samples/s %.2fM'%(d['value']/1e6), 'emb_a2a', round(st['emb_a2a']['ms_per_step'],3), 'nvlink GB/s', round(a['nvlink_gbs_per_gpu'],1))
" $f; done
