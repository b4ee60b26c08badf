export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
A="--no-cpu-baseline --no-e2e --steps 30"
for r in 1 2; do for f in 1 0; do
  NEST_FUSE_REFRESH=$f timeout 300 python bench.py $A > gpurun_out/fr${f}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/fr*_r*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/fr*_r*.json")):
    d=json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    print(f, d["dbp"], d["stages"].get("refresh"))
PY
