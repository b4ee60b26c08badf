export CUDA_VISIBLE_DEVICES=0
A="--no-cpu-baseline --no-e2e --steps 30"
L=$PWD/paper_2604_06956_b200
for r in 1 2; do for n in 16 8 32; do
  lib=$L/libnest.so; [ $n != 16 ] && lib=$L/libnest_ri$n.so
  NEST_LIB=$lib timeout 300 python bench.py $A > gpurun_out/ri${n}_r$r.json 2>/dev/null
done; done
python scripts/bsum.py gpurun_out/ri*_r*.json
B="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-fwp-compare --variant e"
for n in 16 8 32; do
  lib=$L/libnest.so; [ $n != 16 ] && lib=$L/libnest_ri$n.so
  NEST_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_radix|k_scan" --csv python bench.py $B > gpurun_out/ri_ncu_$n.csv 2>/dev/null
  python scripts/launch_table.py gpurun_out/ri_ncu_$n.csv | tail -6
done
