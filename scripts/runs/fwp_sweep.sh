# FWP sweep at W = $W: Zipf skew x micro-batches x schedule,
# the correlated variant, and the tower depth L; summary -> gpurun_out/fwp_sweep_w$W.txt
W=${W:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr 127.0.0.1"
A="--gpus $W --no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
p=29700
out=gpurun_out/fwp_sweep_w$W
mkdir -p $out
run() { tag=$1; shift; p=$((p+1)); timeout 600 $T --master-port $p bench.py $A "$@" > $out/$tag.json 2>/dev/null; }
for z in 0.8 1.05 1.2 1.4; do
  for N in 1 2 4; do
    run z${z}_N${N}_seq --zipf $z --micro-batches $N
    [ $N -gt 1 ] && run z${z}_N${N}_cl --zipf $z --micro-batches $N --schedule clustered-offline
  done
done
for N in 1 2 4; do
  run corr_N${N}_seq --correlated 64,0.5 --micro-batches $N
  [ $N -gt 1 ] && run corr_N${N}_cl --correlated 64,0.5 --micro-batches $N --schedule clustered-offline
done
for L in 2 8; do for N in 1 2; do run L${L}_N${N} --tower-layers $L --micro-batches $N; done; done
python - <<'PY' > gpurun_out/fwp_sweep_w$W.txt
import json, glob, os
W = os.environ.get("W", "2")
print("tag ms/step Msamples/s exposed_a2a_ms physical_a2a_ms exposed_ratio alpha cluster_ms")
for f in sorted(glob.glob(f"gpurun_out/fwp_sweep_w{W}/*.json")):
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception as e:
        print(os.path.basename(f), "failed"); continue
    a = d.get("a2a") or {}
    fw = d["fwp"]
    print(f"{os.path.basename(f)[:-5]:18s} {d['ms_per_step']:.3f} {d['value']/1e6:6.2f} "
          f"{a.get('exposed_ms_per_step', 0):.3f} {a.get('physical_ms_per_step', 0):.3f} "
          f"{(a.get('exposed_ratio') or 0):.3f} {(fw.get('alpha') or 0):.4f} {fw.get('cluster_ms_per_batch')}")
PY
cat gpurun_out/fwp_sweep_w$W.txt
