mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:1:fft 2048:1:fft 4096:1:fft 8192:1:fft"
for i in 1 2; do for v in cur j1 j2; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/j_ab.log
for v in j1; do export PPFG_SO=build/libppfg_$v.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -p no:cacheprovider -x -k "fft or channelize" > gpurun_out/h_parity_$v.log 2>&1; echo $v; tail -1 gpurun_out/h_parity_$v.log; done
