mkdir -p gpurun_out
python scripts/run_op.py --op fft --C 1024 --T 1 --gib 1 --reps 1 > /dev/null && \
ncu --set full --clock-control none -k regex:fft_tiles -c 1 -o gpurun_out/k2n_c1024 -f python scripts/run_op.py --op fft --C 1024 --T 1 --gib 1 --reps 1 > gpurun_out/ncu_k2n.log 2>&1
python scripts/run_op.py --op fir --C 1024 --T 8 --gib 1 --reps 1 > /dev/null && \
ncu --set full --clock-control none -k regex:fir_tma -c 1 -o gpurun_out/k1t_t8 -f python scripts/run_op.py --op fir --C 1024 --T 8 --gib 1 --reps 1 > gpurun_out/ncu_k1t.log 2>&1
tail -1 gpurun_out/ncu_k2n.log gpurun_out/ncu_k1t.log
