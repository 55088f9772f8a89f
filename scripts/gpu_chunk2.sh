mkdir -p gpurun_out
export PPFG_B2B=1
P="1024:8:exact 1024:8:exact-unfused 1024:16:exact-unfused 2048:8:exact-unfused 8192:8:exact 8192:8:fast 1024:32:fast 4096:8:exact"
for c in 0 16 32 64 96; do
  PPFG_UNFUSED_CHUNK_MIB=$c TAG=c$c timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{\|rror'
done > gpurun_out/chunk2.log
