export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --steps 10"
timeout 900 python bench.py --config genrec $A > gpurun_out/cfg_genrec_w1.json 2>gpurun_out/cfg_genrec_w1.err; echo "genrec rc=$?"; tail -2 gpurun_out/cfg_genrec_w1.err
for p in 0.3 0.5 0.7; do
  timeout 900 python bench.py --config dbp_stress --reuse $p $A > gpurun_out/cfg_dbp_stress_p$p.json 2>/dev/null; echo "dbp $p rc=$?"
done
timeout 300 python bench.py --config tiny $A > gpurun_out/cfg_tiny_w1.json 2>/dev/null; echo "tiny rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cfg_*.json")):
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception as e:
        print(f, "failed"); continue
    print(f, round(d["value"]/1e6, 3), "M samples/s", round(d["ms_per_step"], 3), "ms", d["roofline"]["kernel"],
          round(d["roofline"]["frac"], 3), "dbp", {k: d["dbp"][k] for k in ("intersection_ratio", "refresh_ms_per_step")},
          "E", d["embedding_only"] and round(d["embedding_only"]["ms_per_step"], 3))
PY
