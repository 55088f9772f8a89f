# correctness of the variants (fused parity tests through PPFG_SO) + A/B timings
mkdir -p gpurun_out
for v in $1; do
  echo "== $v tests: $(PPFG_SO=build/libppfg_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'fused_vs_oracle or fused_small or tiny or stream_golden' 2>&1 | tail -1)"
done
echo "== cur tests: $(timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'tiny or stream or fused_small' 2>&1 | tail -1)"
bash scripts/gpu_ab2.sh "$1"
