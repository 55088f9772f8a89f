# A/B of register/cluster variants of the EXACT C=1024 T=8 cluster entry (build/libppfg_V.so from build_variant.sh)
mkdir -p gpurun_out
P="1024:8:exact" bash scripts/gpu_variants.sh "r136tw4 q4 q4r152 w4" > gpurun_out/ab1.log 2>&1
P="1024:8:exact" bash scripts/gpu_variants.sh "r136tw4 q4 q4r152 w4" >> gpurun_out/ab1.log 2>&1
cat gpurun_out/ab1.log
