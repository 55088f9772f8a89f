mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-configs > gpurun_out/bench_nc.log 2> gpurun_out/bench_nc.err; tail -1 gpurun_out/bench_nc.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['value'], l['e2e']['value'], l['e2e']['pageable'])"
timeout 300 tools/dropin_loop > gpurun_out/dropin_loop.json 2>&1; cat gpurun_out/dropin_loop.json | cut -c1-300
timeout 300 tools/stream_bench > gpurun_out/stream_bench.json 2>&1; tail -2 gpurun_out/stream_bench.json | cut -c1-300
