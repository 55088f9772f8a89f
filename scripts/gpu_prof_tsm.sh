mkdir -p gpurun_out
export PPFG_SO=build/libppfg_tsm.so
python scripts/run_op.py --op fused --mode exact --C 1024 --T 8 --gib 0.25 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -o gpurun_out/k3_tsm_exact -f python scripts/run_op.py --op fused --mode exact --C 1024 --T 8 --gib 0.25 --reps 1 > gpurun_out/ncu_tsm.log 2>&1
tail -1 gpurun_out/ncu_tsm.log
