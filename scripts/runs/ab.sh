# A/B of bench.py variants on one box, rounds interleaved (the form behind
# every profiles/r02/ab_*.txt).  Usage (through gpurun):
#   bash scripts/runs/ab.sh ROUNDS PREFIX "tag ENV=v ..." "tag ENV=v ..." ... -- [bench.py args]
# e.g.  bash scripts/runs/ab.sh 2 zc "zc0 NEST_ZERO_COPY=0" "zc1 NEST_ZERO_COPY=1" -- --no-e2e --steps 30
#       GPUS=2 bash scripts/runs/ab.sh 2 w2 "chunks NEST_SEGSUM=chunks" "range NEST_SEGSUM=range" -- --variant e
# A tuning build of the library is selected with NEST_LIB=paper_2604_06956_b200/libnest_<tag>.so
# (built with paper_2604_06956_b200/build.py's out= and NEST_NVCC_EXTRA).
# Output: gpurun_out/<PREFIX>_<tag>_r<round>.json, then a bsum.py summary.
set -u
rounds=$1; prefix=$2; shift 2
variants=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do variants+=("$1"); shift; done
[ $# -gt 0 ] && shift
gpus=${GPUS:-1}
port=$((29600 + RANDOM % 300))
for r in $(seq 1 "$rounds"); do
  for v in "${variants[@]}"; do
    read -r tag envs <<< "$v"
    out=gpurun_out/${prefix}_${tag}_r$r.json
    port=$((port + 1))
    if [ "$gpus" -gt 1 ]; then
      env $envs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node="$gpus" \
        --master-addr 127.0.0.1 --master-port $port bench.py --gpus "$gpus" --no-cpu-baseline "$@" > "$out" 2>/dev/null
    else
      env CUDA_VISIBLE_DEVICES=0 $envs timeout 900 python bench.py --no-cpu-baseline "$@" > "$out" 2>/dev/null
    fi
    echo "$tag r$r rc=$?"
  done
done
python scripts/bsum.py gpurun_out/${prefix}_*_r*.json
