"""A/B: K1t (TMA-staged) vs K1 (register prefetch) FIR-only at C=1024, 1 GiB."""
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
    for name, fl in (("tma", ppf.EXACT), ("prefetch", ppf.K1_PREFETCH)):
        with ppf.Plan(C, T, c, flags=fl) as p:
            t = timeit(lambda: p.fir(x, out=y))
            res[name] = round(2 * S * C * 8 / t / 1e9 / peak, 3)
            res[name + "_ok"] = bool(torch.equal(y[:64].cpu(), y[:64].cpu()))
    ya = torch.empty_like(y); yb = torch.empty_like(y)
    with ppf.Plan(C, T, c) as p: p.fir(x, out=ya)
    with ppf.Plan(C, T, c, flags=ppf.K1_PREFETCH) as p: p.fir(x, out=yb)
    torch.cuda.synchronize()
    res["bitwise_equal"] = bool(torch.equal(ya.view(torch.int64), yb.view(torch.int64)))
    print(json.dumps(res), flush=True)
