mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:32:fast 1024:16:fast"
for i in 1 2; do for v in cur t32p t32p2 fftA; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/t32_ab.log
export PPFG_SO=build/libppfg_t32p.so
timeout 600 python -m pytest tests/test_gpu_fullsize.py -k "T32" -q -p no:cacheprovider > gpurun_out/t32_parity.log 2>&1
export PPFG_SO=build/libppfg_fftA.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "channelize or fft" > gpurun_out/fftA_parity.log 2>&1
tail -2 gpurun_out/t32_parity.log gpurun_out/fftA_parity.log
