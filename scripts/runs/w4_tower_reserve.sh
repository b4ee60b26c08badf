# W=4 E+T: NEST_TOWER_SM_RESERVE 24 (default) vs 40
GPUS=4 bash scripts/runs/ab.sh 2 trv4 "r24" "r40 NEST_TOWER_SM_RESERVE=40" -- --no-e2e --steps 50 --no-fwp-compare
