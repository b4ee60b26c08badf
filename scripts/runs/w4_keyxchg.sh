# W=4: key exchange over NCCL (default) vs the window, E and E+T
GPUS=4 bash scripts/runs/ab.sh 2 kx4e "nccl" "win NEST_ROUTE_XCHG=window" -- --no-e2e --steps 30 --no-fwp-compare --variant e
GPUS=4 bash scripts/runs/ab.sh 2 kx4et "nccl" "win NEST_ROUTE_XCHG=window" -- --no-e2e --steps 50 --no-fwp-compare
