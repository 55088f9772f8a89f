# full check: gpu tests, smoke, default bench (with configs), tools
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.log | cut -c1-300; grep "Elapsed\|Maximum resident" gpurun_out/bench_default.err
timeout 300 tools/dropin_loop > gpurun_out/dropin_loop.json 2>&1; cat gpurun_out/dropin_loop.json
timeout 300 tools/dropin_loop 1024 8 1024 1024 >> gpurun_out/dropin_loop.json 2>&1; tail -1 gpurun_out/dropin_loop.json
timeout 300 tools/stream_bench > gpurun_out/stream_bench.json 2>&1; cat gpurun_out/stream_bench.json
timeout 900 tools/ppf_sweep 512 3 > gpurun_out/ppf_sweep.csv 2> gpurun_out/ppf_sweep.jsonl; cat gpurun_out/ppf_sweep.csv
