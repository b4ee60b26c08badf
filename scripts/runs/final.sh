export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -6
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_bench.json 2>gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2>&1; echo "ref rc=$?"
python scripts/bsum.py gpurun_out/final_bench.json
tail -c 400 gpurun_out/final_ref.json
