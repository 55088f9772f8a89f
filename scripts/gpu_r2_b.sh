mkdir -p gpurun_out
SECONDS=0
timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo "bench rc=$? ${SECONDS}s"; tail -1 gpurun_out/bench_default.log | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider 2>&1 | tail -2
MALLOC_MMAP_THRESHOLD_=4294967296 MALLOC_TRIM_THRESHOLD_=8589934592 timeout 300 tools/dropin_loop > gpurun_out/dropin_loop_malloc.json 2>&1; cat gpurun_out/dropin_loop_malloc.json
echo "== shs tests: $(PPFG_SO=build/libppfg_shs.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'fused_vs_oracle or fused_small or mean_power' 2>&1 | tail -1)"
BENCH_ARGS="--mode exact" P="1024:16:fast 1024:8:exact 1024:16:exact 2048:8:fast 2048:8:exact 4096:8:fast 1024:32:fast-cluster 1024:8:detect-exact" bash scripts/gpu_ab2.sh shs
