# direct write-back (sole-contributor keys applied by the requester): parity at
# W = 2 / 4 / 8 ranks on one GPU and over 2 GPUs, then a W=2 A/B (E and E+T)
timeout 1500 python -m pytest tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -3
GPUS=2 bash scripts/runs/ab.sh 2 dwb "on" "off NEST_DIRECT_WB=0" -- --no-e2e --steps 30 --no-fwp-compare --variant e
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/dwb_*.json")):
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception:
        print(f, "failed"); continue
    st = d["stages"]
    print(f, "E ms", round(d["ms_per_step"], 3), "update", round(st["update"]["ms_per_step"], 3),
          "grad_a2a", round(st["grad_a2a"]["ms_per_step"], 3), "whole", round(d["whole_step_hbm"]["frac"], 3))
PY
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29777 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/dwb_w2_bench.json 2>/dev/null
python scripts/bsum.py gpurun_out/dwb_w2_bench.json
