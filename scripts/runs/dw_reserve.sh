# W=1 E+T: SMs left free by the deferred dW GEMMs (NEST_TOWER_DW_SM_RESERVE; the fwd/dX GEMMs keep 24)
bash scripts/runs/ab.sh 2 dwr "r24" "r48 NEST_TOWER_DW_SM_RESERVE=48" "r74 NEST_TOWER_DW_SM_RESERVE=74" "r0 NEST_TOWER_DW_SM_RESERVE=0" -- --no-e2e --steps 50 --no-fwp-compare
