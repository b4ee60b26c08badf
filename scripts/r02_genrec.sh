export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py --config genrec --no-cpu-baseline --steps 10 > gpurun_out/cfg_genrec_w1.json 2>gpurun_out/cfg_genrec_w1.err; echo "genrec rc=$?"; tail -2 gpurun_out/cfg_genrec_w1.err
python scripts/bsum.py gpurun_out/cfg_genrec_w1.json
