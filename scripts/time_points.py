"""Time a few (C, T, mode) points of ppfg_fir_fft / channelize on device-resident
1 GiB inputs; prints one JSON line per point with the HBM roofline fraction
(in + out bytes / time / measured peak). For quick A/B runs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_3656_b200 import ppf
from scripts.sweep import timeit
import bench
peak, _ = bench.measured_peak()
FL = {"fast": ppf.FAST, "exact": ppf.EXACT, "fast-unfused": ppf.FAST | ppf.UNFUSED,
      "fast-cluster": ppf.FAST | ppf.CLUSTER, "exact-unfused": ppf.UNFUSED,
      "fast-l2x": ppf.FAST | ppf.L2X, "exact-l2x": ppf.EXACT | ppf.L2X}
tag = os.environ.get("TAG", "")
for spec in sys.argv[1:]:
    C, T, mode = spec.split(":")
    C, T = int(C), int(T)
    S = (1 << 30) // (C * 8)
    x = torch.empty((S, C), dtype=torch.complex64, device="cuda"); ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device="cuda")
    c = ppf.generate_prototype(C, T)
    if mode in ("detect", "detect-exact"):   # fused FIR+FFT+mean power: input bytes only
        with ppf.Plan(C, T, c, flags=ppf.FAST if mode == "detect" else ppf.EXACT) as p:
            t = timeit(lambda: p.fir_fft_mean_power(x))
        B = S * C * 8
    elif mode == "fir":   # FIR only (bit-exact)
        with ppf.Plan(C, T, c) as p:
            t = timeit(lambda: p.fir(x, out=y))
        B = (2 * S - T + 1) * C * 8
    elif mode in ("fft", "fft-oop"):   # channelize_block, in place / out of place
        z = x if mode == "fft" else torch.empty_like(x)
        with ppf.Plan(C, 1, ppf.generate_prototype(C, 1)) as p:
            t = timeit(lambda: p.channelize(x, out=z))
        B = 2 * S * C * 8
    elif mode == "cufft":
        t = timeit(lambda: torch.fft.fft(x, dim=1))
        B = 2 * S * C * 8
    else:
        with ppf.Plan(C, T, c, flags=FL[mode]) as p:
            t = timeit(lambda: p.fir_fft(x, out=y))
        B = (2 * S - T + 1) * C * 8
    print(json.dumps({"tag": tag, "C": C, "T": T, "mode": mode, "ms": round(t * 1e3, 4),
                      "frac": round(B / t / 1e9 / peak, 4)}), flush=True)
    del x, y
