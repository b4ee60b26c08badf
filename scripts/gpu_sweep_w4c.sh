i=0
run() { # label N env...
  i=$((i+1)); label=$1; N=$2; shift 2
  env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29850+i)) bench.py --gpus 4 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $N > gpurun_out/w4c_${label}_n$N.log 2>&1; echo $label N=$N rc=$?
}
run base 1 NEST_X=0
for N in 2 4; do
  run prio $N NEST_X=0
  run prio_cap192 $N NEST_EMB_MAX_BLOCKS=192
  run prio_cap592 $N NEST_EMB_MAX_BLOCKS=592
  run oldprio $N NEST_LANE_PRIORITIES=0,-1,0
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/w4c_*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); a=d["a2a"]; st=d["stages"]
        print(f.split('/')[-1][4:-4], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | a2a", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "| tower", round(st["tower"]["ms_per_step"],3), "pool", round(st["pool"]["ms_per_step"],3), "emb", round(st["emb_a2a"]["ms_per_step"],3), "grad", round(st["grad_a2a"]["ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
