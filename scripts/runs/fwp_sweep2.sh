# the FWP sweep entries that failed before the bench's per-rank K was all-reduced
W=${W:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr 127.0.0.1"
A="--gpus $W --no-cpu-baseline --no-e2e --no-fwp-compare --steps 20"
p=29900
out=gpurun_out/fwp_sweep_w$W
mkdir -p $out
run() { tag=$1; shift; p=$((p+1)); timeout 600 $T --master-port $p bench.py $A "$@" > $out/$tag.json 2>$out/$tag.err; }
for N in 1 2 4; do
  run z0.8_N${N}_seq --zipf 0.8 --micro-batches $N
  [ $N -gt 1 ] && run z0.8_N${N}_cl --zipf 0.8 --micro-batches $N --schedule clustered-offline
done
run z1.05_N4_seq --micro-batches 4
run z1.05_N4_cl --micro-batches 4 --schedule clustered-offline
run corr_N4_seq --correlated 64,0.5 --micro-batches 4
run corr_N4_cl --correlated 64,0.5 --micro-batches 4 --schedule clustered-offline
# without the early push: the embedding All2All inside the window, where FWP overlaps it
for N in 1 2 4; do NEST_EARLY_PUSH=0 run noep_N${N}_seq --micro-batches $N; done
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
