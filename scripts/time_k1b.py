"""A/B: K1b (register-blocked FIR) vs the lane-window kernels, C=1024, 1 GiB.
FIR-only roofline fraction (in + out bytes / time / peak): exact (FP64) and,
for T >= 32, the FAST unfused FIR+FFT."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_3656_b200 import ppf
from scripts.sweep import timeit
import bench
peak, _ = bench.measured_peak()
C = int(os.environ.get("C", 1024))
for T in [int(t) for t in sys.argv[1].split(",")]:
    S = (1 << 30) // (C * 8)
    x = torch.empty((S, C), dtype=torch.complex64, device="cuda"); ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device="cuda")
    B = (2 * S - T + 1) * C * 8
    res = {"C": C, "T": T}
    c = ppf.generate_prototype(C, T)
    for name, fl in (("k1b", ppf.EXACT), ("legacy", ppf.FIR_LEGACY)):
        with ppf.Plan(C, T, c, flags=fl) as p:
            res["fir_" + name] = round(B / timeit(lambda: p.fir(x, out=y)) / 1e9 / peak, 3)
    for name, fl in (("k1b", ppf.FAST | ppf.UNFUSED), ("legacy", ppf.FAST | ppf.UNFUSED | ppf.FIR_LEGACY),
                     ("default", ppf.FAST)):
        with ppf.Plan(C, T, c, flags=fl) as p:
            res["fast_" + name] = round(B / timeit(lambda: p.fir_fft(x, out=y)) / 1e9 / peak, 3)
    print(json.dumps(res), flush=True)
