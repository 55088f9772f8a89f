# ncu --set full of K1 (FIR only, bit-exact) at C=$1 T=$2
C=${1:-1024}; T=${2:-32}
mkdir -p gpurun_out
python scripts/run_op.py --op fir --C $C --T $T > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fir_chain -s 1 -c 1 -f -o gpurun_out/prof_fir_${C}_${T} python scripts/run_op.py --op fir --C $C --T $T > gpurun_out/ncu_f.log 2>&1
ncu -i gpurun_out/prof_fir_${C}_${T}.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_fir_${C}_${T}_src.csv 2>/dev/null
tail -1 gpurun_out/ncu_f.log
