# ncu --set full of the bench's dominant kernel at the bench's own config (SKA, C=1024 T=8 FAST)
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_fir_fft -s 2 -c 1 -f -o gpurun_out/prof_bench python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
ncu -i gpurun_out/prof_bench.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_bench_src.csv 2>/dev/null
tail -2 gpurun_out/ncu_b.log
