mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:16:fast"
for i in 1 2; do for v in cur t16a t16b t16c t16d; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/t16_ab.log
