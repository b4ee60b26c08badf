set -x
i=0
for cfg in "16 16 4" "32 32 4" "64 0 4" "32 32 1" "64 0 1"; do
  set -- $cfg; i=$((i+1))
  NEST_NCCL_MAX_CTAS=$1 NEST_TOWER_SM_RESERVE=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches $3 > gpurun_out/sweep_$1_$2_$3.log 2>&1
  echo "cfg=$cfg rc=$?"
done
NEST_NCCL_MAX_CTAS=64 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 2 --steps 30 --warmup 3 --no-e2e --no-fwp-compare --micro-batches 1 --variant e > gpurun_out/sweep_e_n1.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/sweep_*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l)
        a=d["a2a"]; print(f, round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms a2a_phys", round(a["physical_ms_per_step"],3), "exp", round(a["exposed_ms_per_step"],3), "GB/s", round(a["nvlink_gbs_per_gpu"],1), "tower", round(d["stages"].get("tower",{}).get("ms_per_step",0),3))
    except Exception as e: print(f, "err", e)
PY
export CUDA_VISIBLE_DEVICES=0
CMD="python bench.py --variant e --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_e.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_e.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:segsum_cold -s 8 -c 2 -o gpurun_out/prof_segsum $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
