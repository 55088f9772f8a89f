timeout 300 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider -k "stream or refsuite" 2>&1 | tail -1
echo "new $(timeout 200 python scripts/time_push.py)"
cp paper_1411_3656_b200/libppfg.so build/libppfg_cur.so; cp build/libppfg_old.so paper_1411_3656_b200/libppfg.so; touch paper_1411_3656_b200/libppfg.so
echo "old $(timeout 200 python scripts/time_push.py)"
cp build/libppfg_cur.so paper_1411_3656_b200/libppfg.so; touch paper_1411_3656_b200/libppfg.so
