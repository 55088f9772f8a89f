# A/B of register/cluster/twiddle variants of cluster entries (build/libppfg_V.so from build_variant.sh)
mkdir -p gpurun_out
for i in 1 2; do
P="1024:32:fast-cluster 1024:32:fast" bash scripts/gpu_variants.sh "t32r136 t32r168 t32q8" >> gpurun_out/ab1.log 2>&1
done
cat gpurun_out/ab1.log
