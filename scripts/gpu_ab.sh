# A/B: the working-tree library vs build/libppfg_old.so on the same points (+ SKA bench)
mkdir -p gpurun_out
P=${P:-"1024:8:fast 512:8:fast 1024:1:fft"}
TAG=new python scripts/time_points.py $P 2>&1 | grep '^{'
python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150
cp paper_1411_3656_b200/libppfg.so build/libppfg_new.so; cp build/libppfg_old.so paper_1411_3656_b200/libppfg.so
TAG=old python scripts/time_points.py $P 2>&1 | grep '^{'
python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150
cp build/libppfg_new.so paper_1411_3656_b200/libppfg.so
