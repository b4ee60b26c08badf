# DBP stress (refresh at rising batch overlap) and the FWP sweep (Zipf skew x
# micro-batches x clustering, + correlated samples), W=2.  Summary ->
# gpurun_out/sweep_summary.txt
i=0
run() { # tag args...
  i=$((i+1)); tag=$1; shift
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29700+i)) bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --no-fwp-compare "$@" > gpurun_out/sw_$tag.log 2>&1
  echo "$tag rc=$?"
}
for p in 0.2 0.45 0.7; do run dbp_p$p --config dbp_stress --reuse $p --variant e; done
for z in 0.8 1.05 1.4; do
  run fwp_z${z}_n1 --zipf $z --micro-batches 1
  for N in 2 4; do for S in sequential clustered; do run fwp_z${z}_n${N}_$S --zipf $z --micro-batches $N --schedule $S; done; done
done
for S in sequential clustered; do run corr_n4_$S --correlated 64,0.5 --micro-batches 4 --schedule $S; done
# generative-rec sequence feature (unpooled, embedding-only), W=2 and W=1
run genrec_w2 --config genrec --steps 10
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config genrec --steps 10 --warmup 3 --no-e2e --no-fwp-compare --no-cpu-baseline > gpurun_out/sw_genrec_w1.log 2>&1; echo "genrec_w1 rc=$?"
python - <<'PY' > gpurun_out/sweep_summary.txt
import json,glob
print("| run | samples/s (M) | ms/step | a2a physical ms | a2a exposed ms | exposed ratio | alpha (sum_i U_i / U) | schedule ms | refresh ms | I / U_o | tower ms |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob("gpurun_out/sw_*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"] or {}; st=d["stages"]; fw=d["fwp"]; db=d["dbp"]
        print(f"| {f.split('/')[-1][3:-4]} | {d['value']/1e6:.2f} | {d['ms_per_step']:.3f} | {a.get('physical_ms_per_step',0):.3f} | {a.get('exposed_ms_per_step',0):.3f} | {(a.get('exposed_ratio') or 0):.2f} | {fw['alpha']:.3f} | {st.get('schedule',{}).get('ms_per_step',0):.3f} | {db['refresh_ms_per_step']:.3f} | {(db['intersection_ratio'] or 0):.3f} | {st.get('tower',{}).get('ms_per_step',0):.3f} |")
    except Exception as e: print("|", f, "err", e, "|")
PY
cat gpurun_out/sweep_summary.txt
