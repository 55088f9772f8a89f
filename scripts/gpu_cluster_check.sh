mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -p no:cacheprovider -k "cluster or small_and_ragged" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
timeout 300 python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import torch
from scripts.sweep import timeit
from paper_1411_3656_b200 import ppf
import bench
peak, _ = bench.measured_peak()
for C, T, fl in [(2048, 8, ppf.FAST), (1024, 16, ppf.FAST), (1024, 8, ppf.EXACT), (4096, 8, ppf.FAST), (8192, 8, ppf.FAST), (1024, 32, ppf.FAST), (1024, 16, ppf.EXACT), (2048, 8, ppf.EXACT)]:
    S = (1 << 30) // (C * 8)
    x = torch.empty((S, C), dtype=torch.complex64, device='cuda'); ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device='cuda')
    c = ppf.generate_prototype(C, T)
    res = []
    for f in (fl | ppf.CLUSTER, fl | ppf.UNFUSED):
        with ppf.Plan(C, T, c, flags=f) as p:
            t = timeit(lambda: p.fir_fft(x, out=y))
            res.append((p.kind, round(2 * S * C * 8 / t / 1e9 / peak, 3)))
    print(C, T, fl, res, flush=True)
PY
