# segment-sum range length R: in-step time (E, E+T) and ncu DRAM traffic per launch
export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
L=paper_2604_06956_b200
for r in 1 2; do
for R in 256 128 64; do
  lib=$L/libnest.so; [ $R != 256 ] && lib=$PWD/$L/libnest_r$R.so
  NEST_LIB=$lib timeout 300 python bench.py $A > gpurun_out/rng${R}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/rng*_r*.json
B="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare --variant e"
for R in 256 128 64; do
  lib=$L/libnest.so; [ $R != 256 ] && lib=$PWD/$L/libnest_r$R.so
  NEST_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"k_segsum" -s 6 -c 6 --csv python bench.py $B > gpurun_out/rng_ncu_$R.csv 2>/dev/null
  echo "R=$R"; grep -E "k_segsum" gpurun_out/rng_ncu_$R.csv | awk -F'","' '{print $5" "$(NF-2)" "$(NF-1)" "$NF}' | cut -c1-160 | head -12
done
