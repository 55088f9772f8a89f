"""Time the SKA step (C=1024, T=8, 793,464 input spectra = 6.5 GB, FAST and
EXACT) and cfg1 back to back on device-resident data: one JSON line per run
(A/B of library variants via PPFG_SO)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1411_3656_b200 import ppf
import bench
peak, _ = bench.measured_peak()
tag = os.environ.get("TAG", "")
for (C, T, S, mode) in ((1024, 8, 793464, "fast"), (512, 8, 131072, "fast")):
    x = torch.empty((S, C), dtype=torch.complex64, device="cuda")
    ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device="cuda")
    c = ppf.generate_prototype(C, T)
    with ppf.Plan(C, T, c, flags=ppf.FAST if mode == "fast" else ppf.EXACT) as p:
        for _ in range(3):
            p.fir_fft(x, out=y)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        ev = []
        for _ in range(8):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); p.fir_fft(x, out=y); b.record(s); ev.append((a, b))
        torch.cuda.synchronize()
        t = float(np.median([a.elapsed_time(b) for a, b in ev[1:]])) / 1e3
        name = p.kernel_name
    B = 8 * C * (2 * S - T + 1)
    print(json.dumps({"tag": tag, "C": C, "T": T, "S": S, "mode": mode, "ms": round(t * 1e3, 4),
                      "in_gbps": round(8 * C * S / t / 1e9, 1), "frac": round(B / t / 1e9 / peak, 4),
                      "kernel": name[:90]}), flush=True)
    del x, y
