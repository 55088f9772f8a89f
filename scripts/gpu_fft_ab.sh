mkdir -p gpurun_out
timeout 300 python scripts/host_overhead.py > gpurun_out/host_overhead.json 2>&1
P="64:1:fft 128:1:fft 256:1:fft 512:1:fft 1024:1:fft 2048:1:fft"
for i in 1 2; do for v in cur fftA fftB; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/fft_ab.log
