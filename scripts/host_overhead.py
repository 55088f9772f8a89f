"""Host-side cost of one library call and its effect on single-launch CUDA-event
timing: per-call host time (small input, Python + ctypes + library), and the
1 GiB C=1024 T=8 FAST launch timed (a) rep-by-rep with a sync in between (the
host's submission gap inside the events) and (b) back-to-back (gap hidden)."""
import json
import time
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1411_3656_b200 import ppf, _lib

dev = torch.device("cuda:0")
res = {}
for (C, T, fl, name) in ((1024, 8, ppf.FAST, "k3_fast"), (1024, 8, ppf.EXACT, "k3s_exact"),
                         (1024, 32, ppf.FAST, "unfused_t32")):
    coeffs = ppf.generate_prototype(C, T)
    with ppf.Plan(C, T, coeffs, flags=fl) as p:
        x = torch.empty((64, C), dtype=torch.complex64, device=dev)
        ppf.synth(C, 64 * C, seed=1, out=x)
        y = torch.empty((64 - T + 1, C), dtype=torch.complex64, device=dev)
        for _ in range(20):
            p.fir_fft(x, out=y)
        torch.cuda.synchronize()
        n = 2000
        t0 = time.perf_counter()
        for _ in range(n):
            p.fir_fft(x, out=y)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        res[name + "_host_us_per_call_python"] = (t1 - t0) / n * 1e6
        # raw ctypes, no Python wrapper work
        lib = _lib.load()
        h = p.handle
        st = torch.cuda.current_stream().cuda_stream
        fn = lib.ppfg_fir_fft_device if hasattr(lib, "ppfg_fir_fft_device") else None
        S = 1 << 30
        S_in = S // (C * 8)
        X = torch.empty((S_in, C), dtype=torch.complex64, device=dev)
        ppf.synth(C, S_in * C, seed=2, out=X)
        Y = torch.empty((S_in - T + 1, C), dtype=torch.complex64, device=dev)
        for _ in range(3):
            p.fir_fft(X, out=Y)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        sy = []
        for _ in range(7):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); p.fir_fft(X, out=Y); b.record(s); torch.cuda.synchronize()
            sy.append(a.elapsed_time(b))
        ev = []
        for _ in range(7):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); p.fir_fft(X, out=Y); b.record(s); ev.append((a, b))
        torch.cuda.synchronize()
        bb = [a.elapsed_time(b) for a, b in ev]
        # a sleep kernel ahead of the start event hides the submission gap
        sl = []
        for _ in range(7):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)
            a.record(s); p.fir_fft(X, out=Y); b.record(s); torch.cuda.synchronize()
            sl.append(a.elapsed_time(b))
        res[name + "_1GiB_ms"] = {"synced": float(np.median(sy)), "back_to_back": float(np.median(bb[1:])),
                                  "after_sleep": float(np.median(sl)), "kernel": p.kernel_name}
        del X, Y
print(json.dumps(res, indent=1))
