# split re-push (sole-contributor keys re-pushed as soon as their writer's flag arrives): parity + W=2 A/B
timeout 1500 python -m pytest tests/test_gpu_local_ranks.py -q -x 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "fused-early or no-nccl" 2>&1 | tail -2
GPUS=2 bash scripts/runs/ab.sh 2 srE "split" "whole NEST_EARLY_REPUSH=0" -- --no-e2e --steps 30 --no-fwp-compare --variant e
GPUS=2 bash scripts/runs/ab.sh 3 srET "split" "whole NEST_EARLY_REPUSH=0" -- --no-e2e --steps 50 --no-fwp-compare
