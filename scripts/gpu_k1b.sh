mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x -k "fir_block or fir_bitwise or fused_vs_oracle" > gpurun_out/pytest_k1b.log 2>&1; tail -3 gpurun_out/pytest_k1b.log
timeout 900 python scripts/time_k1b.py ${1:-16,24,32,48,64,96,128} 2>&1 | tail -8
