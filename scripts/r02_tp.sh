export CUDA_VISIBLE_DEVICES=0
timeout 1500 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -6
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/r02_profile.sh
