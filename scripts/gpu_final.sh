# end-of-session refresh: all GPU tests, smoke, bench lines, sweep, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-200
timeout 300 python bench.py --steps 5 --warmup 3 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_ska_exact.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --config cfg1 --no-e2e > gpurun_out/bench_cfg1_fast.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --config cfg1 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_exact.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --config long16 --no-e2e --no-cpu-baseline --spectra 1000000 > gpurun_out/bench_long16.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 1200 python scripts/sweep.py --md gpurun_out/sweep.md > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 ./tools/stream_bench 1024 8 2048 4096 > gpurun_out/stream_bench.json 2>&1; cat gpurun_out/stream_bench.json
echo done
