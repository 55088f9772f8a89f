mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:32:fast"
for i in 1 2; do for v in cur w4a w4b; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/ts_ab.log
export PPFG_SO=build/libppfg_w4b.so
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_guards.py -k "T32 or 1024-32 or K1b" -q -p no:cacheprovider -x > gpurun_out/ts_parity.log 2>&1; tail -3 gpurun_out/ts_parity.log
