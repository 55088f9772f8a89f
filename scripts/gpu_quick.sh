# quick loop: GPU parity tests + SKA bench + cfg1 bench + one ncu --set full of the fused kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ska_fast.log 2>&1; tail -1 gpurun_out/bench_ska_fast.log | cut -c1-600
python bench.py --steps 10 --warmup 3 --config cfg1 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_fast.log 2>&1
python bench.py --steps 10 --warmup 3 --config cfg1 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_exact.log 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --spectra 200000 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/prof_fused -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --spectra 200000 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
