mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "mean_power" 2>&1 | tail -2
timeout 300 python scripts/time_points.py 1024:8:detect 1024:8:detect-exact 512:8:detect 2048:8:detect 1024:16:detect 256:8:detect 2>&1 | grep '^{'
