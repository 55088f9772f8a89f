mkdir -p gpurun_out
python scripts/sweep.py --md gpurun_out/sweep.md > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; tail -3 gpurun_out/sweep.err
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/sweep.md
