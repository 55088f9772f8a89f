mkdir -p gpurun_out
export PPFG_B2B=1
P="512:8:fast 128:8:fast 64:8:fast 512:16:fast"
for i in 1 2 3; do for v in cur tr1; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/tr1_ab.log
export PPFG_SO=build/libppfg_tr1.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "fused or guard or cfg1 or chan or power or ragged" > gpurun_out/tr1_parity.log 2>&1; tail -1 gpurun_out/tr1_parity.log
