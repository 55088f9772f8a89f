mkdir -p gpurun_out
for i in 1 2; do for v in cur il8 il16 il32 il64; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_ska.py 2>&1 | grep '^{\|rror'
done; done > gpurun_out/il_ab.log
export PPFG_SO=build/libppfg_il16.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "fused or power or cfg1 or guard or special or ragged or small" > gpurun_out/il_parity.log 2>&1; tail -1 gpurun_out/il_parity.log
