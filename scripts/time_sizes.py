"""fir_fft throughput by input size (device-resident, back to back): does the
rate drop for multi-GB streams? usage: time_sizes.py C T mode GB..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1411_3656_b200 import ppf
import bench
peak, _ = bench.measured_peak()
C, T, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
pad = int(os.environ.get("PAD_ROWS", "0"))   # output view offset (address aliasing probe)
for gb in [float(g) for g in sys.argv[4:]]:
    S = int(gb * 1e9) // (C * 8)
    x = torch.empty((S, C), dtype=torch.complex64, device="cuda")
    ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1 + pad, C), dtype=torch.complex64, device="cuda")[pad:]
    with ppf.Plan(C, T, ppf.generate_prototype(C, T), flags=ppf.FAST if mode == "fast" else ppf.EXACT) as p:
        p.fir_fft(x, out=y)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        ev = []
        for _ in range(4):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); p.fir_fft(x, out=y); b.record(s); ev.append((a, b))
        torch.cuda.synchronize()
        t = float(np.median([a.elapsed_time(b) for a, b in ev[1:]])) / 1e3
    B = 8 * C * (2 * S - T + 1)
    print(json.dumps({"C": C, "T": T, "mode": mode, "GB": gb, "pad_rows": pad, "ms": round(t * 1e3, 3),
                      "frac": round(B / t / 1e9 / peak, 4)}), flush=True)
    del x, y
    torch.cuda.empty_cache()
