#!/usr/bin/env python
"""Taps sweep (C=1024, T=4..64) and channels sweep (T=8, C=64..8192) on one
B200, 1 GiB of input per point (BASELINE.json configs 3 and 4).

Per point, device-resident, CUDA events on the launch stream, median of 5
after 2 warm-ups:
  fused_fast  ppfg_fir_fft, PPFG_FAST   (fused FP32-FIR kernel where one exists)
  exact       ppfg_fir_fft, PPFG_EXACT  (bit-exact: fused FP64 or FIR->FFT)
  fir         ppfg_fir (K1, bit-exact FP64 accumulation) alone
  fft         ppfg_channelize (K2, bit-exact radix-2) alone, in place
  cufft       torch.fft.fft over the same rows (cuFFT; comparison point only)
  detect      ppfg_fir_fft_mean_power, PPFG_FAST (per-channel mean power; frac =
              input bytes / time / peak, the pass being read-only when fused)
GB/s = input bytes / time; roofline frac = (in + out bytes) / time / peak.
Writes JSON lines to stdout and a markdown table to --md.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1411_3656_b200 import ppf  # noqa: E402
import bench  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    s = torch.cuda.current_stream()
    if os.environ.get("PPFG_B2B"):   # back to back: the host's submission gap hidden
        ev = []
        for _ in range(reps + 1):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            ev.append((a, b))
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ev[1:]])) / 1e3
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def point(C, T, gib, peak):
    S = max(T, (int(gib * (1 << 30))) // (C * 8))
    dev = torch.device("cuda:0")
    x = torch.empty((S, C), dtype=torch.complex64, device=dev)
    ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device=dev)
    coeffs = ppf.generate_prototype(C, T)
    bin_, bout = S * C * 8, (S - T + 1) * C * 8
    res = {"C": C, "T": T, "S_in": S, "bytes_in": bin_}
    for mode, flags in (("fused_fast", ppf.FAST), ("exact", ppf.EXACT)):
        with ppf.Plan(C, T, coeffs, flags=flags) as p:
            t = timeit(lambda: p.fir_fft(x, out=y))
            res[mode] = {"ms": t * 1e3, "gbs_in": bin_ / t / 1e9,
                         "frac": (bin_ + bout) / t / 1e9 / peak,
                         "kernel": ["unfused", "fused-fp32", "fused-fp64", "cluster-fp32", "cluster-fp64", "tiny-fp32", "tiny-fp64", "l2x-fp32", "l2x-fp64"][p.kind]}
    with ppf.Plan(C, T, coeffs, flags=ppf.FAST) as p:
        # detection (mean power per channel): only the input is HBM traffic
        # when a fused detection kernel exists
        t = timeit(lambda: p.fir_fft_mean_power(x))
        res["detect"] = {"ms": t * 1e3, "gbs_in": bin_ / t / 1e9, "frac": bin_ / t / 1e9 / peak}
    with ppf.Plan(C, T, coeffs) as p:
        t = timeit(lambda: p.fir(x, out=y))
        res["fir"] = {"ms": t * 1e3, "gbs_in": bin_ / t / 1e9,
                      "frac": (bin_ + bout) / t / 1e9 / peak}
        t = timeit(lambda: p.channelize(y, out=y))
        res["fft"] = {"ms": t * 1e3, "frac": 2 * bout / t / 1e9 / peak}
    t = timeit(lambda: torch.fft.fft(y, dim=1))
    res["cufft"] = {"ms": t * 1e3, "frac": 2 * bout / t / 1e9 / peak}
    del x, y
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--md", default="")
    ap.add_argument("--which", default="taps,channels")
    args = ap.parse_args()
    peak, src = bench.measured_peak()
    pts = []
    if "taps" in args.which:
        pts += [(1024, t) for t in (4, 8, 16, 32, 64)]
    if "channels" in args.which:
        pts += [(c, 8) for c in (64, 128, 256, 512, 1024, 2048, 4096, 8192)]
    rows = []
    for C, T in pts:
        r = point(C, T, args.gib, peak)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if args.md:
        with open(args.md, "w") as f:
            f.write(f"# Sweep ({args.gib} GiB input per point, HBM peak {peak} GB/s {src})\n\n")
            f.write("| C | T | fused FAST GB/s in (frac, kernel) | EXACT GB/s in (frac, kernel) | "
                    "FIR-only GB/s in (frac) | FFT-only ms (frac) | cuFFT ms (frac) | "
                    "detect FAST GB/s in (frac of read-only) |\n")
            f.write("|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['C']} | {r['T']} | {r['fused_fast']['gbs_in']:.0f} "
                        f"({r['fused_fast']['frac']:.2f}, {r['fused_fast']['kernel']}) | "
                        f"{r['exact']['gbs_in']:.0f} ({r['exact']['frac']:.2f}, "
                        f"{r['exact']['kernel']}) | {r['fir']['gbs_in']:.0f} ({r['fir']['frac']:.2f})"
                        f" | {r['fft']['ms']:.3f} ({r['fft']['frac']:.2f}) | "
                        f"{r['cufft']['ms']:.3f} ({r['cufft']['frac']:.2f}) | "
                        f"{r['detect']['gbs_in']:.0f} ({r['detect']['frac']:.2f}) |\n")


if __name__ == "__main__":
    main()
