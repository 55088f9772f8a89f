# final evidence: launch list + ncu --set full of the timed SKA kernel (FAST) and
# the EXACT sub-record kernel, cfg1, and the K6 / C=4096 / long16 kernels
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact --no-configs"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_fir_fft -s 2 -c 1 -f -o gpurun_out/k3_ska_final $B > gpurun_out/ncu_full.log 2>&1; echo "ska rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fused_split -s 2 -c 1 -f -o gpurun_out/k3s_ska_exact_final python bench.py --steps 2 --warmup 3 --mode exact --no-e2e --no-cpu-baseline --no-parity --no-configs > gpurun_out/ncu_full2.log 2>&1; echo "exact rc=$?"
ncu --set full --clock-control none --import-source on -k regex:fused_fir_fft -s 2 -c 1 -f -o gpurun_out/k3_cfg1_final python bench.py --config cfg1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact --no-configs > gpurun_out/ncu_full3.log 2>&1; echo "cfg1 rc=$?"
ncu --set full --clock-control none -k regex:fused_split -s 2 -c 1 -f -o gpurun_out/k3s_c4096_final python scripts/time_points.py 4096:8:fast > gpurun_out/ncu_full4.log 2>&1; echo "c4096 rc=$?"
ncu --set full --clock-control none -k regex:fused_tiny -s 2 -c 1 -f -o gpurun_out/k6_c8_final python scripts/time_points.py 8:8:fast > gpurun_out/ncu_full5.log 2>&1; echo "tiny rc=$?"
