"""Debug: phase timeline of CTA 0 of the split cluster kernel (needs the
-DPPFG_TRACE build selected with PPFG_SO)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1411_3656_b200 import ppf, _lib
C_, T = int(sys.argv[1]), int(sys.argv[2])
flags = ppf.FAST if len(sys.argv) < 4 else int(sys.argv[3])
S = (256 << 20) // (C_ * 8)
x = torch.empty((S, C_), dtype=torch.complex64, device="cuda"); ppf.synth(C_, S * C_, seed=3, out=x)
y = torch.empty((S - T + 1, C_), dtype=torch.complex64, device="cuda")
with ppf.Plan(C_, T, ppf.generate_prototype(C_, T), flags=flags | ppf.CLUSTER) as p:
    for _ in range(2):
        p.fir_fft(x, out=y)
    torch.cuda.synchronize()
buf = np.zeros(2 * 16 * 64, np.uint64)
_lib.load().ppfg_debug_trace(C.c_void_p(buf.ctypes.data))
buf = buf.reshape(2, 16, 64).astype(np.int64)
t0 = buf[:, :8][buf[:, :8] > 0].min()
names = {0: ["start", "empty_ok", "ring_ok", "stored", "issued"], 1: ["start", "local_ok", "remote_ok", "done"]}
ev = []
for role in (0, 1):
    for e, nm in enumerate(names[role]):
        for b in range(64):
            if buf[role, e, b] > 0:
                ev.append((buf[role, e, b] - t0, ["fir", "fft"][role], b, nm))
ev.sort()
for t, r, b, nm in ev[:160]:
    print(f"{t/1000:9.3f} us {r} b={b:2d} {nm}")
