"""Generate tests/golden/*.npz from the UNMODIFIED reference, compiled from
/root/reference by oracle/Makefile (oracle/_ref). Run in the build container:

    python tests/golden/make_golden.py

Inputs are the reference tests' own distributions (uniform [-1, 1], mt19937
is replaced by numpy's PCG64 with fixed seeds; the values themselves are
stored, so no generator needs to match). Outputs are exactly what the
reference returns. The fixtures are small (< 2 MB total) and travel with the
repo; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def uni(rng, n):
    return rng.uniform(-1.0, 1.0, size=2 * n).astype(np.float32)


def main():
    R = oracle.reference()
    if R is None:
        raise SystemExit("oracle/_ref not available (needs /root/reference)")
    rng = np.random.default_rng(20141113)
    out = {}

    # FIR: reference shapes (fir_test.cpp:136-169, acceptance_test.cpp:121-153)
    fir = []
    for C, T, extra in [(1, 1, 5), (2, 2, 3), (8, 4, 20), (8, 8, 6), (64, 8, 12), (1024, 16, 4),
                        (256, 32, 3), (3, 5, 9), (16, 64, 2), (1024, 8, 9)]:
        S = T + extra
        x = uni(rng, S * C)
        c = R.generate_prototype(C, T, 9.0)
        fir.append(dict(C=C, T=T, x=x, coeffs=c, y=R.fir(x, C, T, c, reference=False, workers=3),
                        y_ref=R.fir(x, C, T, c, reference=True)))
    # impulse (fir_test.cpp:87-110): exact zeros and signed zeros
    C, T, S = 4, 5, 12
    x = np.zeros(S * C * 2, np.float32)
    x[2 * (6 * C + 2)] = 1.0
    c = rng.uniform(0.25, 1.75, C * T) * np.where(rng.uniform(size=C * T) < 0.5, -1, 1)
    fir.append(dict(C=C, T=T, x=x, coeffs=c, y=R.fir(x, C, T, c), y_ref=R.fir(x, C, T, c,
                                                                               reference=True)))
    for i, f in enumerate(fir):
        for k, v in f.items():
            out[f"fir{i}_{k}"] = v
    out["n_fir"] = len(fir)

    # FFT / channelize: every power of two 1..8192, plus dft_naive sizes
    ns = [1 << k for k in range(14)]
    for n in ns:
        rows = max(1, 4096 // n) if n < 4096 else 2
        x = uni(rng, rows * n)
        out[f"fft{n}_x"] = x
        out[f"fft{n}_y"] = R.channelize(x, n, True, workers=2)
    out["fft_sizes"] = np.array(ns)
    dn = [3, 5, 6, 7, 12, 100, 127, 1000]
    for n in dn:
        x = uni(rng, 2 * n)
        out[f"dft{n}_x"] = x
        out[f"dft{n}_y"] = R.channelize(x, n, True)
    out["dft_sizes"] = np.array(dn)

    # fused one-shot (pipeline_test.cpp:40-51 one_shot): FIR then channelize
    fused = []
    for C, T, S in [(512, 8, 40), (1024, 8, 24), (64, 8, 100), (256, 4, 30), (16, 4, 300),
                    (6, 3, 20)]:
        x = uni(rng, S * C)
        c = R.generate_prototype(C, T, 9.0)
        fused.append(dict(C=C, T=T, x=x, coeffs=c, y=R.fir_fft(x, C, T, c, True, workers=2)))
    for i, f in enumerate(fused):
        for k, v in f.items():
            out[f"ff{i}_{k}"] = v
    out["n_ff"] = len(fused)

    # prototype spot shapes (coeff_test.cpp:191-209) incl. rectangular
    protos = [(4, 8, 9.0), (16, 4, 6.5), (3, 7, 0.0), (64, 8, 9.0), (1024, 8, 9.0), (512, 16, 9.0)]
    for i, (C, T, b) in enumerate(protos):
        out[f"proto{i}"] = R.generate_prototype(C, T, b)
    out["protos"] = np.array(protos)

    # streaming: C=8, T=8, 2500 spectra + 3 trailing samples (pipeline_test.cpp:156-170,
    # 203-217); stream output is block-size invariant
    C, T, S = 8, 8, 2500
    x = uni(rng, S * C + 3)
    src = x.tobytes()
    c = R.generate_prototype(C, T, 9.0)
    y, st = R.process_stream(src, C, T, 100, c)
    out["stream_x"] = np.frombuffer(src, np.uint8)
    out["stream_y"] = np.frombuffer(y, np.uint8)
    out["stream_state"] = np.array([st.spectra_processed, st.bytes_in, st.bytes_out,
                                    st.dropped_samples], np.uint64)
    yz, stz = R.process_stream(src, C, T, 64, c, zero_prime=True)
    out["stream_zp_y"] = np.frombuffer(yz, np.uint8)
    out["stream_zp_state"] = np.array([stz.spectra_processed, stz.bytes_in, stz.bytes_out,
                                       stz.dropped_samples], np.uint64)
    out["reference_build"] = np.array(os.path.basename(R.path))

    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_vectors.npz"))


if __name__ == "__main__":
    main()
