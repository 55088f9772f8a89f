# gpu_ab2.sh "V1 V2 ..." : SKA bench (with whole-output FAST parity) for the
# working tree ("cur") and build/libppfg_V.so variants, twice, + 1 GiB points P
mkdir -p gpurun_out
P=${P:-"1024:8:fast"}
cp paper_1411_3656_b200/libppfg.so build/libppfg_cur.so
for i in 1 2; do
for v in cur $1; do
  cp build/libppfg_$v.so paper_1411_3656_b200/libppfg.so; touch paper_1411_3656_b200/libppfg.so
  echo "== $v bench: $(timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-exact $BENCH_ARGS 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); p=d.get("parity") or {}; print(round(d["value"],1), round(d["roofline"]["frac"],4), "parity", p.get("pass"), p.get("max_err_over_rms"))')"
  TAG=$v timeout 300 python scripts/time_points.py $P 2>&1 | grep '^{'
done; done
cp build/libppfg_cur.so paper_1411_3656_b200/libppfg.so; touch paper_1411_3656_b200/libppfg.so
