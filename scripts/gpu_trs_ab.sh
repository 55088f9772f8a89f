mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:16:fast 2048:8:fast 4096:8:fast"
for i in 1 2 3; do for v in head trs; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/trs_ab.log
export PPFG_SO=build/libppfg_trs.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "fused or guard or long16 or chan or taps or power" > gpurun_out/trs_parity.log 2>&1; tail -1 gpurun_out/trs_parity.log
