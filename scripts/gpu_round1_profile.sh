set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ska_fast.log 2>&1; tail -1 gpurun_out/bench_ska_fast.log
python bench.py --steps 5 --warmup 3 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_ska_exact.log 2>&1; tail -1 gpurun_out/bench_ska_exact.log
python bench.py --steps 10 --warmup 3 --config cfg1 --no-e2e > gpurun_out/bench_cfg1_fast.log 2>&1; tail -1 gpurun_out/bench_cfg1_fast.log
python bench.py --steps 10 --warmup 3 --config cfg1 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_exact.log 2>&1; tail -1 gpurun_out/bench_cfg1_exact.log
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --spectra 200000 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --spectra 200000 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
