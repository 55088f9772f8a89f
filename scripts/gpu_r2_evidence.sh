# round-2 evidence: launch list of the bench, ncu --set full of the bench's
# dominant kernel, compute-sanitizer racecheck / synccheck / memcheck logs
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_fir_fft -s 2 -c 1 -f -o gpurun_out/k3_ska \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-exact > gpurun_out/ncu_full.log 2>&1
echo "ncu_full rc=$?"
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_kernels.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
