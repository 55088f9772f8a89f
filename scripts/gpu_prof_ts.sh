mkdir -p gpurun_out
python scripts/run_op.py --op fused --mode fast --C 1024 --T 32 --gib 0.25 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_split -c 1 -o gpurun_out/k3s_ts32 -f python scripts/run_op.py --op fused --mode fast --C 1024 --T 32 --gib 0.25 --reps 1 > gpurun_out/ncu_ts32.log 2>&1
tail -1 gpurun_out/ncu_ts32.log
