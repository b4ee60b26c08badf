T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 900 $T --master-port 29711 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/w2_final_bench.json 2>/dev/null
timeout 900 $T --master-port 29712 bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-fwp-compare --micro-batches 2 --variant e > gpurun_out/w2_final_e_n2.json 2>/dev/null
python scripts/bsum.py gpurun_out/w2_final_bench.json gpurun_out/w2_final_e_n2.json
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/w2_final_bench.json").read().splitlines() if l.startswith("{")][-1])
print({k:(round(v["ms_per_step"],3), round(v.get("a2a_exposed_ms_per_step",0),3)) for k,v in d["a2a"]["with_tower"].items()})
PY
