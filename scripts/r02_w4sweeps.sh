# 4-GPU session: gen-rec and DBP stress at W=2/4, FWP sweep subset at W=4
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
T2="env CUDA_VISIBLE_DEVICES=0,1 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--no-cpu-baseline --no-e2e --steps 10"
out=gpurun_out/w4s; mkdir -p $out
p=29900
run() { tag=$1; shift; p=$((p+1)); timeout 900 "$@" > $out/$tag.json 2>$out/$tag.err; echo "$tag rc=$?"; }
run genrec_w2 $T2 --master-port $((p+100)) bench.py --gpus 2 $A --config genrec
run genrec_w4 $T4 --master-port $((p+101)) bench.py --gpus 4 $A --config genrec
for r in 0.3 0.7; do
  run dbp_w4_p$r $T4 --master-port $((p+110)) bench.py --gpus 4 $A --config dbp_stress --reuse $r --no-fwp-compare
done
for N in 1 2 4; do
  run fwp_w4_N$N $T4 --master-port $((p+120+N)) bench.py --gpus 4 $A --no-fwp-compare --micro-batches $N
done
run fwp_w4_N4_cl $T4 --master-port $((p+130)) bench.py --gpus 4 $A --no-fwp-compare --micro-batches 4 --schedule clustered-offline
run fwp_w4_corr_N4_seq $T4 --master-port $((p+131)) bench.py --gpus 4 $A --no-fwp-compare --micro-batches 4 --correlated 64,0.5
run fwp_w4_corr_N4_cl $T4 --master-port $((p+132)) bench.py --gpus 4 $A --no-fwp-compare --micro-batches 4 --correlated 64,0.5 --schedule clustered-offline
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/w4s/*.json")):
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception:
        print(os.path.basename(f), "failed"); continue
    a = d.get("a2a") or {}
    print(f"{os.path.basename(f)[:-5]:22s} {d['n_gpus']} {d['value']/1e6:7.2f}M {d['ms_per_step']:.3f}ms "
          f"exposed {a.get('exposed_ms_per_step', 0):.3f} phys {a.get('physical_ms_per_step', 0):.3f} "
          f"nvl {a.get('nvlink_gbs_per_gpu', 0) or 0:.0f} alpha {d['fwp'].get('alpha')} "
          f"refresh {d['dbp']['refresh_ms_per_step']:.3f} I/Uo {d['dbp']['intersection_ratio']}")
PY
