mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:1:fft 1024:1:cufft"
for i in 1 2; do for v in head cur; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/once_ab.log
unset PPFG_SO
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -p no:cacheprovider -x -k "fft or channelize" > gpurun_out/once_parity.log 2>&1; tail -1 gpurun_out/once_parity.log
