mkdir -p gpurun_out
export PPFG_B2B=1
P="64:1:cufft 1024:1:cufft 8192:1:cufft 1024:1:fft 1024:1:fft-oop 64:1:fft 64:1:fft-oop 1024:8:fast 8192:1:fft"
for i in 1 2; do for v in cur fftA; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/fft_ab2.log
