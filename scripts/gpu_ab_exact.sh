# A/B of register/cluster/twiddle variants (build/libppfg_V.so from build_variant.sh)
mkdir -p gpurun_out
for i in 1 2; do
P="1024:16:fast" bash scripts/gpu_variants.sh "t16_128 t16_144" >> gpurun_out/ab1.log 2>&1
P="1024:4:fast" bash scripts/gpu_variants.sh "t4_136 t4_152" >> gpurun_out/ab1.log 2>&1
done
cat gpurun_out/ab1.log
