# W=2 lane priorities: the owner update (comm lane) vs the DBP lookahead's early push (aux lane)
GPUS=2 bash scripts/runs/ab.sh 2 prE "base" "c5 NEST_LANE_PRIORITIES=-2,-5,0" "c5a4 NEST_LANE_PRIORITIES=-2,-5,0 NEST_AUX_PRIORITY=-4" -- --no-e2e --steps 30 --no-fwp-compare --variant e
GPUS=2 bash scripts/runs/ab.sh 2 prET "base" "c5 NEST_LANE_PRIORITIES=-2,-5,0" "c5a4 NEST_LANE_PRIORITIES=-2,-5,0 NEST_AUX_PRIORITY=-4" -- --no-e2e --steps 30 --no-fwp-compare
