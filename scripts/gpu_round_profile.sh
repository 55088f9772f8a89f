# round profile refresh: bench lines, launch list, ncu full captures of the
# hot kernel (K3 SKA) and the kernels added this session (K1b, K2r), sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ska_fast.log 2>&1; tail -1 gpurun_out/bench_ska_fast.log | cut -c1-200
python bench.py --steps 5 --warmup 3 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_ska_exact.log 2>&1
python bench.py --steps 10 --warmup 3 --config cfg1 --no-e2e > gpurun_out/bench_cfg1_fast.log 2>&1
python bench.py --steps 10 --warmup 3 --config cfg1 --mode exact --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg1_exact.log 2>&1
python bench.py --steps 5 --warmup 3 --config long16 --no-e2e --no-cpu-baseline --spectra 1000000 > gpurun_out/bench_long16.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused -s 1 -c 1 -o gpurun_out/k3_fused_ska -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fir_block -c 1 -o gpurun_out/k1b_fast_t64 -f python scripts/run_op.py --op fused --mode fast-unfused --C 1024 --T 64 --gib 0.5 --reps 1 > gpurun_out/ncu_k1b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fft_ring -c 1 -o gpurun_out/k2r_fft_c8192 -f python scripts/run_op.py --op fft --C 8192 --T 8 --gib 0.5 --reps 1 > gpurun_out/ncu_k2r.log 2>&1
python scripts/sweep.py --md gpurun_out/sweep.md > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
ls gpurun_out
