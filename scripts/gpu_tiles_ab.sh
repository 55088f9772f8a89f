mkdir -p gpurun_out
export PPFG_B2B=1
P="4096:1:fft 4096:8:exact"
for i in 1 2; do for v in cur u1 u2 u3; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/tiles_ab7.log
