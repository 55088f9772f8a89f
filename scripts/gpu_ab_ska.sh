# A/B of the SKA fused entry: the working-tree library ("cur") vs build/libppfg_V.so, SKA bench + 1 GiB point
mkdir -p gpurun_out
cp paper_1411_3656_b200/libppfg.so build/libppfg_cur.so
for i in 1 2; do
for v in cur ${1:-s104 s128 sl2a2}; do
  cp build/libppfg_$v.so paper_1411_3656_b200/libppfg.so
  echo "$v $(python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["frac"],4))')"
  TAG=$v python scripts/time_points.py 1024:8:fast 2>&1 | grep '^{'
done; done
cp build/libppfg_cur.so paper_1411_3656_b200/libppfg.so
