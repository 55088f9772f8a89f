mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:8:fir 1024:4:fir 8192:8:fast 8192:8:exact 1024:32:fast 1024:64:fast 1024:32:exact 1024:16:fir 1024:32:fir"
for i in 1 2; do for v in head cur kb256 kb512 kb1024; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/k1_ab3.log
