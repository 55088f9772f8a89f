mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:8:fast 1024:8:detect 1024:4:fast 512:8:exact 1024:4:exact"
for i in 1 2; do for v in head vt1 vt2; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/vt_ab.log
for v in vt1 vt2; do
export PPFG_SO=build/libppfg_$v.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "fused or power or cfg1 or guard or taps or special" > gpurun_out/vt_parity_$v.log 2>&1; echo $v; tail -1 gpurun_out/vt_parity_$v.log
done
