# k_reduce_sgd: lane-parallel contribution resolution (new) vs serial (old); W=2 A/B
L=$PWD/paper_2604_06956_b200
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mb or micro or N2 or N4 or adagrad or zero" 2>&1 | tail -2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
A="--gpus 2 --no-cpu-baseline --no-e2e --steps 30 --no-fwp-compare --variant e"
p=29620
for r in 1 2; do for v in new old; do
  p=$((p+1)); lib=$L/libnest.so; [ $v = old ] && lib=$L/libnest_rsold.so
  NEST_LIB=$lib timeout 600 $T --master-port $p bench.py $A > gpurun_out/rsab_${v}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/rsab_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/rsab_*.json")):
    d=json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    st=d["stages"]
    print(f, "ms", round(d["ms_per_step"],3), "update", round(st["update"]["ms_per_step"],3), round(st["update"].get("frac_of_measured_hbm",0),3),
          "whole", round(d["whole_step_hbm"]["frac"],3), d["whole_step_hbm"]["stages"])
PY
timeout 900 $T --master-port 29690 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/rs_w2_bench.json 2>/dev/null
python scripts/bsum.py gpurun_out/rs_w2_bench.json
