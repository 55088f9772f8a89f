# gpu_variants.sh "V1 V2 ..." : time points P with the working-tree library ("cur")
# and each build/libppfg_V.so
mkdir -p gpurun_out
P=${P:-"1024:8:fast"}
cp paper_1411_3656_b200/libppfg.so build/libppfg_cur.so
for v in cur $1; do
  cp build/libppfg_$v.so paper_1411_3656_b200/libppfg.so
  TAG=$v python scripts/time_points.py $P 2>&1 | grep '^{'
done
cp build/libppfg_cur.so paper_1411_3656_b200/libppfg.so
