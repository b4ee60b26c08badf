# W=2 E+T: SMs the tower's GEMMs leave to the sparse lanes (NEST_TOWER_SM_RESERVE, default 24)
GPUS=2 bash scripts/runs/ab.sh 2 trv "r24" "r40 NEST_TOWER_SM_RESERVE=40" "r56 NEST_TOWER_SM_RESERVE=56" -- --no-e2e --steps 50 --no-fwp-compare
