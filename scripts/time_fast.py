"""FAST fir_fft at C=1024 for T list: default kernel vs forced unfused (K1f + FFT)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_3656_b200 import ppf
from scripts.sweep import timeit
import bench
peak, _ = bench.measured_peak()
C = 1024
for T in [int(t) for t in sys.argv[1].split(",")]:
    S = (1 << 30) // (C * 8)
    x = torch.empty((S, C), dtype=torch.complex64, device="cuda"); ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device="cuda")
    res = {"T": T}
    c = ppf.generate_prototype(C, T)
    for name, fl in (("default", ppf.FAST), ("unfused", ppf.FAST | ppf.UNFUSED)):
        with ppf.Plan(C, T, c, flags=fl) as p:
            t = timeit(lambda: p.fir_fft(x, out=y))
            res[name] = (p.kind, round(2 * S * C * 8 / t / 1e9 / peak, 3))
    print(json.dumps(res), flush=True)
