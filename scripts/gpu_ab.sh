# A/B: the working-tree library vs build/libppfg_old.so on the same points
mkdir -p gpurun_out
P=${P:-"1024:8:fast 1024:16:fast 1024:32:fast 1024:32:fast-unfused 2048:8:fast 2048:8:exact 4096:8:fast 4096:8:fast-unfused 8192:8:fast 8192:8:fast-cluster 1024:16:exact 1024:8:exact"}
TAG=new python scripts/time_points.py $P 2>&1 | grep '^{'
cp paper_1411_3656_b200/libppfg.so build/libppfg_new.so; cp build/libppfg_old.so paper_1411_3656_b200/libppfg.so
TAG=old python scripts/time_points.py $P 2>&1 | grep '^{'
cp build/libppfg_new.so paper_1411_3656_b200/libppfg.so
