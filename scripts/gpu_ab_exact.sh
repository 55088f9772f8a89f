# A/B of register/cluster/twiddle variants (build/libppfg_V.so from build_variant.sh)
mkdir -p gpurun_out
for i in 1 2; do
P="512:8:exact" bash scripts/gpu_variants.sh "e512_136 e512_144 e512_152 e512_168" >> gpurun_out/ab1.log 2>&1
done
cat gpurun_out/ab1.log
