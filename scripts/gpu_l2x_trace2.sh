for v in cur dbg3 dbg1 u16; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  for pt in 1024:16:fast-l2x 1024:32:fast-l2x; do
    PPFG_L2X_TRACE=gpurun_out/tr_${v}_${pt//:/_}.bin TAG=$v timeout 300 python scripts/time_points.py $pt 2>&1 | grep '^{\|rror'
  done
done
