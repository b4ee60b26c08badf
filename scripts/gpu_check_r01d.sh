export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hot or realistic or dlrm or bit_exact" 2>&1 | tail -3
for C in 32 128 512; do for N in 1 4; do
  NEST_SEG_CHUNK=$C timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches $N --variant e > gpurun_out/d_c${C}_n$N.log 2>&1
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/d_c*_n*.log")):
    try:
        l=[x for x in open(f) if x.startswith("{")][-1]; d=json.loads(l); st=d["stages"]
        print(f.split('/')[-1], round(d["value"]/1e6,2), "Msps", round(d["ms_per_step"],3), "ms | segsum", round(st["segsum"]["ms_per_step"],3), round(st["segsum"]["frac_of_measured_hbm"],2), "pool", round(st["pool"]["ms_per_step"],3))
    except Exception as e: print(f, "err", e)
PY
CMD="python bench.py --variant e --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --micro-batches 4"
$CMD > gpurun_out/plain_d.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_d.csv $CMD > gpurun_out/ncu_d.log 2>&1; echo ncu=$?
