# evidence of the final SKA kernel: launch list + ncu --set full (traffic), and
# ncu summaries of the other headline kernels (EXACT SKA, cfg1, long16, C=8192 unfused)
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact --no-configs"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_fir_fft -s 2 -c 1 -f -o gpurun_out/k3_ska_r2 $B > gpurun_out/ncu_full.log 2>&1; echo "ska rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fused_split -s 2 -c 1 -f -o gpurun_out/k3s_ska_exact_r2 python bench.py --steps 2 --warmup 3 --mode exact --no-e2e --no-cpu-baseline --no-parity --no-configs > gpurun_out/ncu_full2.log 2>&1; echo "exact rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fused_fir_fft -s 2 -c 1 -f -o gpurun_out/k3_cfg1_r2 python bench.py --config cfg1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact --no-configs > gpurun_out/ncu_full3.log 2>&1; echo "cfg1 rc=$?"
