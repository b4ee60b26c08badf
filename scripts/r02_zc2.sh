export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py > gpurun_out/zc_default.json 2>gpurun_out/zc_default.err; echo rc=$?; tail -2 gpurun_out/zc_default.err
python scripts/bsum.py gpurun_out/zc_default.json
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "zero_copy or refresh_required or misuse" 2>&1 | tail -2
