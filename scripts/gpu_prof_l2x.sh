mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_l2x -s 2 -c 1 -f -o gpurun_out/l2x_t32 python scripts/time_points.py 1024:32:fast-l2x > gpurun_out/ncu_l2x.log 2>&1; echo rc=$?; tail -3 gpurun_out/ncu_l2x.log
