#!/bin/bash
# build_variant.sh NAME 'sed-expression' : build libppfg.so from a copy of csrc with
# the fused table edited by the sed expression, into build/libppfg_NAME.so (A/B runs)
set -e
name=$1; expr=$2
d=$(mktemp -d)
cp -r paper_1411_3656_b200/csrc $d/
sed -i "$expr" $d/csrc/*.cu $d/csrc/*.cuh
diff -r paper_1411_3656_b200/csrc $d/csrc | head -20 || true
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared -Iinclude -o build/libppfg_$name.so $d/csrc/ppfg.cu
rm -rf $d
