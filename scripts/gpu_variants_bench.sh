# gpu_variants_bench.sh "V1 V2": SKA bench value + points P for the working tree and variants
mkdir -p gpurun_out
P=${P:-"1024:8:fast"}
cp paper_1411_3656_b200/libppfg.so build/libppfg_cur.so
for v in cur $1; do
  cp build/libppfg_$v.so paper_1411_3656_b200/libppfg.so; touch paper_1411_3656_b200/libppfg.so
  echo "== $v bench: $(timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["frac"],4))')"
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{'
done
cp build/libppfg_cur.so paper_1411_3656_b200/libppfg.so; touch paper_1411_3656_b200/libppfg.so
