mkdir -p gpurun_out
python scripts/run_op.py --op fused --C 2048 --T 8 --mode cluster > gpurun_out/plain_c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_cluster -s 1 -c 1 -f -o gpurun_out/prof_cluster python scripts/run_op.py --op fused --C 2048 --T 8 --mode cluster > gpurun_out/ncu_c.log 2>&1
ncu -i gpurun_out/prof_cluster.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_cluster_src.csv 2>/dev/null
tail -2 gpurun_out/ncu_c.log
