mkdir -p gpurun_out
for T in 8 16; do
python scripts/run_op.py --op fir --T $T > gpurun_out/plain_fir$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fir_chain -s 1 -c 1 -f -o gpurun_out/prof_fir_t$T python scripts/run_op.py --op fir --T $T > gpurun_out/ncu_fir$T.log 2>&1
done
python scripts/run_op.py --op fft > gpurun_out/plain_fft.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fft_rows -s 1 -c 1 -f -o gpurun_out/prof_fft python scripts/run_op.py --op fft > gpurun_out/ncu_fft.log 2>&1
for r in prof_fir_t8 prof_fir_t16 prof_fft; do ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_src.csv 2>/dev/null; done
ls gpurun_out
