for v in cur dbg1 dbg2; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; fi
  echo "== $v"; timeout 300 python scripts/time_points.py 1024:16:fast-l2x 1024:32:fast-l2x 8192:8:fast-l2x 2>&1 | grep '^{\|rror'
done
