# the other BASELINE configs with the final build: W=1 (gen-rec, DBP stress p=0.3/0.5/0.7, tiny) and W=2 (DBP stress p=0.7, gen-rec)
CUDA_VISIBLE_DEVICES=0 bash scripts/runs/configs.sh
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 900 $T2 --master-port 29831 bench.py --gpus 2 --no-cpu-baseline --config dbp_stress --reuse 0.7 --steps 10 > gpurun_out/cfg_w2_dbp_stress_p0.7.json 2>/dev/null; echo "w2 dbp rc=$?"
timeout 900 $T2 --master-port 29832 bench.py --gpus 2 --no-cpu-baseline --config genrec --steps 10 > gpurun_out/cfg_w2_genrec.json 2>/dev/null; echo "w2 genrec rc=$?"
python scripts/bsum.py gpurun_out/cfg_w2_*.json
