export CUDA_VISIBLE_DEVICES=0
for f in chunks range; do for np in "1 1" "1 0" "2 1"; do NEST_SEGSUM=$f python scripts/ada_debug.py $np 2>&1 | tail -1; done; done
