mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "l2x" 2>&1 | tail -5
timeout 300 python scripts/time_points.py 1024:32:fast-l2x 1024:32:fast 1024:64:fast-l2x 1024:64:fast 1024:16:fast-l2x 1024:16:fast 1024:32:exact-l2x 1024:32:exact 8192:8:fast-l2x 8192:8:fast 8192:8:exact-l2x 2>&1 | grep '^{\|Error\|error'
