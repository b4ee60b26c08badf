# W=2 segment-sum form with the current defaults: chunked (W>1 default) vs range
GPUS=2 bash scripts/runs/ab.sh 2 sf "chunks" "range NEST_SEGSUM=range" -- --no-e2e --steps 30 --no-fwp-compare --variant e
GPUS=2 bash scripts/runs/ab.sh 2 sfet "chunks" "range NEST_SEGSUM=range" -- --no-e2e --steps 50 --no-fwp-compare
