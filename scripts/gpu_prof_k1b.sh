mkdir -p gpurun_out
python scripts/run_op.py --op fir --mode exact --C 1024 --T 64 --gib 0.25 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:fir_block -c 1 -o gpurun_out/k1b_exact_t64 -f python scripts/run_op.py --op fir --mode exact --C 1024 --T 64 --gib 0.25 --reps 1 > gpurun_out/ncu_k1b_e.log 2>&1
python scripts/run_op.py --op fused --mode fast-unfused --C 1024 --T 64 --gib 0.25 --reps 1 && \
ncu --set full --clock-control none --import-source on -k regex:fir_block -c 1 -o gpurun_out/k1b_fast_t64 -f python scripts/run_op.py --op fused --mode fast-unfused --C 1024 --T 64 --gib 0.25 --reps 1 > gpurun_out/ncu_k1b_f.log 2>&1
tail -2 gpurun_out/ncu_k1b_e.log gpurun_out/ncu_k1b_f.log
