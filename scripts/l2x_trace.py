"""Print K7's CTA-0 timeline dumped by PPFG_L2X_TRACE (u64 [2 roles][8][256] ns)."""
import sys
import numpy as np
tr = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(2, 8, 256).astype(np.int64)
t0 = tr[tr > 0].min()
f = lambda a: np.where(a > 0, (a - t0) / 1000.0, np.nan)   # us
fir, fft = f(tr[0]), f(tr[1])
print("FIR items (us): start, +spin(consumed), +barrier, +wait-first-chunk, compute-end")
for m in range(0, 40):
    if np.isnan(fir[0, m]):
        break
    print(f"  item {m:3d}: {fir[0,m]:8.2f}  spin {fir[1,m]-fir[0,m]:6.2f}  bar {fir[2,m]-fir[1,m]:6.2f}"
          f"  tma {fir[4,m]-fir[3,m]:6.2f}  compute {fir[5,m]-fir[4,m]:6.2f}  total {fir[0,m+1]-fir[0,m] if m+1 < 256 else 0:6.2f}")
for g in (0, 1):
    print(f"FFT group {g} tiles (us): start, wait(produced), passes")
    for i in range(0, 60):
        if np.isnan(fft[2 * g, i]):
            continue
        print(f"  tile {i:3d}: {fft[2*g,i]:8.2f}  wait {fft[2*g+1,i]-fft[2*g,i]:7.2f}  passes {fft[4+g,i]-fft[2*g+1,i]:6.2f}")
