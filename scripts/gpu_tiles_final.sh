mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
export PPFG_B2B=1
P="64:1:fft 128:1:fft 256:1:fft 512:1:fft 1024:1:fft 2048:1:fft 4096:1:fft 1024:32:fast 1024:64:fast 1024:32:exact 4096:8:exact 100:4:exact"
for i in 1 2; do for v in head cur; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/tiles_final.log
