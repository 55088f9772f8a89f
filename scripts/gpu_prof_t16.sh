mkdir -p gpurun_out
python scripts/run_op.py --op fused --mode fast --C 1024 --T 16 --gib 0.5 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_split -c 1 -o gpurun_out/k3s_t16 -f python scripts/run_op.py --op fused --mode fast --C 1024 --T 16 --gib 0.5 --reps 1 > gpurun_out/ncu_t16.log 2>&1
tail -1 gpurun_out/ncu_t16.log
