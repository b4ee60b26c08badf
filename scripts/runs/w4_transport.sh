# W=4 transport A/B (E step): fused SM stores (default) vs copy engines vs fused + copy-engine early push
GPUS=4 bash scripts/runs/ab.sh 2 w4t "fused" "ce NEST_A2A=ce" "epce NEST_EARLY_PUSH=ce" -- --no-e2e --steps 30 --no-fwp-compare --variant e
for f in gpurun_out/w4t_*.json; do python -c "
import json,sys
f=sys.argv[1]
d=json.loads([l for l in open(f).read().splitlines() if l.startswith('{')][-1])
a=d['a2a']
print(f.split('/')[-1], 'E ms', round(d['ms_per_step'],3), 'a2a phys', round(a['physical_ms_per_step'],3), 'exposed', round(a['exposed_ms_per_step'],3), 'nvlink GB/s', round(a['nvlink_gbs_per_gpu'],1))
" $f; done
