mkdir -p gpurun_out
for v in cur cvA cvB; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -k "special_values or fused_vs_oracle" -q -p no:cacheprovider > gpurun_out/special_$v.log 2>&1; echo $v; tail -1 gpurun_out/special_$v.log
done
export PPFG_B2B=1
P="1024:8:exact 512:8:exact 64:8:exact 1024:4:exact 1024:16:exact 2048:8:exact"
for i in 1 2; do for v in head cur cvA cvB; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/f2f_ab.log
