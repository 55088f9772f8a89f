mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:32:fast 1024:64:fast 4096:32:fast"
for i in 1 2; do for v in cur ffa ffa2; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/fb_ab.log
for v in ffa ffa2; do
export PPFG_SO=build/libppfg_$v.so
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_parity.py -k "T32 or T64 or K1b or fast" -q -p no:cacheprovider -x > gpurun_out/ffa_parity_$v.log 2>&1; tail -1 gpurun_out/ffa_parity_$v.log
done
