for pt in 1024:16:fast-l2x 1024:32:fast-l2x; do
  PPFG_L2X_TRACE=gpurun_out/tr_${pt//:/_}.bin timeout 300 python scripts/time_points.py $pt 2>&1 | grep '^{\|rror'
done
