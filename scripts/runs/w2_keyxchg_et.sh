# W=2 E+T: key exchange over NCCL (default) vs the window, 3 rounds
GPUS=2 bash scripts/runs/ab.sh 3 kxet "nccl" "win NEST_ROUTE_XCHG=window" -- --no-e2e --steps 50 --no-fwp-compare
