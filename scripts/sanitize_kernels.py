"""One small launch of every kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck): K3 fused FP32 and FP64, K3s cluster
kernels (FP32 T=16, FP64 T=8, C=4096), K1b FIR (T=64), K2n (C=8192), the T=1
fused FFT, K4 dft_naive, detection. Each result is also checked against the
oracle so a run under the sanitizer is a correctness run too.

    compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1411_3656_b200 import ppf  # noqa: E402

port = oracle.port()
CASES = [  # (C, T, flags, S_in)
    (1024, 8, ppf.FAST, 160),                     # K3 SKA shape
    (512, 8, ppf.EXACT, 120),                     # K3 FP64
    (1024, 16, ppf.FAST, 60),                     # K3s 2-CTA cluster FP32
    (1024, 8, ppf.EXACT, 60),                     # K3s FP64
    (4096, 8, ppf.FAST, 24),                      # K3s C = 4096
    (1024, 64, ppf.FAST, 200),                    # K1b FP32 + T=1 fused FFT
    (256, 64, ppf.EXACT, 150),                    # K1b FP64 + K3 T=1
    (8192, 8, ppf.FAST, 12),                      # K1t + K2n
    (100, 4, ppf.EXACT, 40),                      # K1 + K4 dft_naive
]
for C, T, flags, S in CASES:
    x = ppf.synth(C, S * C, seed=C + T)
    c = port.generate_prototype(C, T, 9.0)
    with ppf.Plan(C, T, c, flags=flags) as p:
        y = p.fir_fft(x)
        name = p.kernel_name
        pw = p.fir_fft_mean_power(x)
    want = port.fir_fft(x, C, T, c).view(np.complex64).reshape(-1, C)
    if flags & ppf.FAST:
        w = want.astype(np.complex128)
        err = np.abs(y.astype(np.complex128) - w).max() / np.sqrt(np.mean(np.abs(w) ** 2))
        ok = err <= 1e-5 * np.log2(C)
    else:
        ok = np.array_equal(y.view(np.uint32), want.view(np.uint32))
    pw_want = port.mean_power(want, C)
    ok_pw = np.allclose(pw, pw_want, rtol=1e-4 if flags & ppf.FAST else 1e-12, atol=0)
    print(f"C={C} T={T} {'FAST' if flags & ppf.FAST else 'EXACT'} S={S}: {name} "
          f"fir_fft {'ok' if ok else 'MISMATCH'}, detection {'ok' if ok_pw else 'MISMATCH'}",
          flush=True)
    assert ok and ok_pw
print("all kernel families ran")
