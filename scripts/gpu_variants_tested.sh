# gpu_variants_tested.sh "V1 V2" "pytest -k expr": for each build/libppfg_V.so run the
# selected GPU tests (bounded) and time points P; then restore the working-tree library
mkdir -p gpurun_out
P=${P:-"1024:8:fast"}
cp paper_1411_3656_b200/libppfg.so build/libppfg_cur.so
for v in cur $1; do
  cp build/libppfg_$v.so paper_1411_3656_b200/libppfg.so
  touch paper_1411_3656_b200/libppfg.so
  if [ -n "$2" ] && [ "$v" != cur ]; then
    echo "== tests $v: $(timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -p no:cacheprovider -k "$2" 2>&1 | tail -1)"
  fi
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{'
done
cp build/libppfg_cur.so paper_1411_3656_b200/libppfg.so
touch paper_1411_3656_b200/libppfg.so
