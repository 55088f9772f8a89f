mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:8:exact"
for i in 1 2; do for v in cur f3a f3b f2w4; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/f3_ab.log
export PPFG_SO=build/libppfg_f3a.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -p no:cacheprovider -x -k "fused or guard or special" > gpurun_out/f3_parity.log 2>&1; tail -1 gpurun_out/f3_parity.log
