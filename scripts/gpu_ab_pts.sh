# A/B of 1 GiB points only: cur (in-tree) vs build/libppfg_V.so, twice
for i in 1 2; do for v in cur $1; do
  if [ $v != cur ]; then export PPFG_SO=build/libppfg_$v.so; else unset PPFG_SO; fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done; done
