mkdir -p gpurun_out
export PPFG_B2B=1
P="4096:1:fft 8192:1:fft 8192:8:fast"
for i in 1 2; do for v in cur g1 g2; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/g_ab.log
