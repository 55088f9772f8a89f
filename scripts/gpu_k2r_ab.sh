mkdir -p gpurun_out
export PPFG_B2B=1
P="8192:1:fft 8192:1:cufft 8192:8:fast 8192:8:exact"
for i in 1 2; do for v in cur r3g r2g; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/k2r_ab.log
export PPFG_SO=build/libppfg_r3g.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py -k "fft or 8192 or ring" -q -p no:cacheprovider > gpurun_out/k2r_parity.log 2>&1; tail -1 gpurun_out/k2r_parity.log
