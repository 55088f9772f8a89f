mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "l2x" 2>&1 | tail -2
timeout 300 python scripts/time_points.py 1024:32:fast-l2x 1024:64:fast-l2x 1024:16:fast-l2x 1024:32:exact-l2x 8192:8:fast-l2x 8192:8:exact-l2x 2>&1 | grep '^{\|Error\|error'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_l2x -s 2 -c 1 -f -o gpurun_out/l2x_t16 python scripts/time_points.py 1024:16:fast-l2x > gpurun_out/ncu_l2x.log 2>&1; echo rc=$?
