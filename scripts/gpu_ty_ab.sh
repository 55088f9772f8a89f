mkdir -p gpurun_out
export PPFG_B2B=1
P="8:8:fast 8:8:exact 32:16:fast 1:8:fast 1:4:fast 2:4:exact 16:8:exact"
for i in 1 2; do for v in cur ty8 ty32; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done > gpurun_out/ty_ab.log
