# ncu --set full of the split cluster kernel at C=$1 T=$2 (default 1024 16)
C=${1:-1024}; T=${2:-16}
mkdir -p gpurun_out
python scripts/run_op.py --op fused --C $C --T $T --mode cluster > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_split -s 1 -c 1 -f -o gpurun_out/prof_split_${C}_${T} python scripts/run_op.py --op fused --C $C --T $T --mode cluster > gpurun_out/ncu_s.log 2>&1
ncu -i gpurun_out/prof_split_${C}_${T}.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_split_${C}_${T}_src.csv 2>/dev/null
tail -2 gpurun_out/ncu_s.log
