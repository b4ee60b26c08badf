# W=2 E step: the route's key exchange (count AllGather + key All2All) over NCCL (default) vs the window; NCCL CTA cap
GPUS=2 bash scripts/runs/ab.sh 2 kx "nccl" "win NEST_ROUTE_XCHG=window" "cta32 NEST_NCCL_MAX_CTAS=32" -- --no-e2e --steps 30 --no-fwp-compare --variant e
for f in gpurun_out/kx_*.json; do python -c "
import json,sys
f=sys.argv[1]
d=json.loads([l for l in open(f).read().splitlines() if l.startswith('{')][-1]); st=d['stages']
print(f.split('/')[-1], 'E ms', round(d['ms_per_step'],3), 'key_a2a', round(st.get('key_a2a',{}).get('ms_per_step',0),3), 'update', round(st['update']['ms_per_step'],3), 'emb_a2a', round(st['emb_a2a']['ms_per_step'],3))
" $f; done
