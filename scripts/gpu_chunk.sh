for mb in 0 16 32 64 128; do
  echo "== chunk $mb MB"; PPFG_CHUNK_MB=$mb timeout 300 python scripts/time_points.py 1024:32:fast 1024:64:fast 1024:32:exact 1024:64:exact 8192:8:fast 8192:8:exact 2>&1 | grep '^{\|rror'
done
