mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x -k "fir_block or fir_bitwise or fused_vs_oracle" > gpurun_out/pytest_k1b.log 2>&1; tail -3 gpurun_out/pytest_k1b.log
timeout 600 python scripts/time_k1b.py 16,32,64,128 2>&1 | tail -6
