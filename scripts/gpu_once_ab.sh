mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:1:fft 1024:1:cufft"
for i in 1 2; do for v in cur ca cc cd ce cf; do
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/once_ab2.log
