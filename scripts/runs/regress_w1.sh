# W=1 regression check: the current tree vs an older checkout in _prev/ (git worktree), interleaved
export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 50 --no-fwp-compare ${VARIANT:+--variant $VARIANT}"
for r in 1 2 3; do
  timeout 300 python bench.py $A > gpurun_out/rg_cur_r$r.json 2>/dev/null
  (cd _prev && timeout 300 python bench.py $A > ../gpurun_out/rg_prev_r$r.json 2>/dev/null)
done
python scripts/bsum.py gpurun_out/rg_*.json
