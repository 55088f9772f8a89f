mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -p no:cacheprovider -k "l2x or L2 or K7" 2>&1 | tail -2
for pt in 1024:16:fast-l2x 1024:32:fast-l2x 1024:64:fast-l2x 1024:32:exact-l2x 8192:8:fast-l2x 8192:8:exact-l2x; do
  PPFG_L2X_TRACE=gpurun_out/tr_v2_${pt//:/_}.bin timeout 300 python scripts/time_points.py $pt 2>&1 | grep '^{\|rror'
done
