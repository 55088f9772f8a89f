mkdir -p gpurun_out
export PPFG_B2B=1
P="512:8:fast 512:8:exact 1024:8:fast 1024:1:fft 64:1:fft 256:8:fast 1024:4:fast"
for i in 1 2; do for v in head cur; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
  TAG=$v timeout 300 python scripts/time_ska.py 2>&1 | grep '^{\|rror'
done; done > gpurun_out/pdl_ab.log
unset PPFG_SO
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
