mkdir -p gpurun_out
for T in 32 64; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active --clock-control none --csv python scripts/run_op.py --op fused --mode fast --C 1024 --T $T --gib 1 --reps 1 > gpurun_out/unf_t$T.csv 2>&1
done
