mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:8:exact 1024:16:fast 2048:8:fast"
for i in 1 2; do for v in cur tsm; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/tsm_ab.log
export PPFG_SO=build/libppfg_tsm.so
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/tsm_parity.log 2>&1; tail -3 gpurun_out/tsm_parity.log
