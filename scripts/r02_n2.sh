export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
A="--no-cpu-baseline --no-e2e --steps 30 --micro-batches 2 --variant e --no-fwp-compare"
for r in 1 2; do timeout 300 python bench.py $A > gpurun_out/n2fold_r$r.json 2>/dev/null; done
python scripts/bsum.py gpurun_out/n2fold_r*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/n2fold_r*.json")):
    d=json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1]); print(f, d["stages"]["sort"])
PY
