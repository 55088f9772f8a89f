#!/usr/bin/env python
"""Run one library op a few times on device-resident synthetic input — the
command line ncu wraps to profile a single kernel.

  python scripts/run_op.py --op fir|fft|fused|unfused --C 1024 --T 8 [--gib 1] [--mode fast|exact]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_3656_b200 import ppf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="fir")
    ap.add_argument("--C", type=int, default=1024)
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--mode", default="exact")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    C, T = a.C, a.T
    S = int(a.gib * (1 << 30)) // (C * 8)
    dev = torch.device("cuda:0")
    x = torch.empty((S, C), dtype=torch.complex64, device=dev)
    ppf.synth(C, S * C, seed=3, out=x)
    y = torch.empty((S - T + 1, C), dtype=torch.complex64, device=dev)
    flags = {"fast": ppf.FAST, "exact": ppf.EXACT, "unfused": ppf.UNFUSED,
             "cluster": ppf.FAST | ppf.CLUSTER, "exact-cluster": ppf.CLUSTER,
             "fast-unfused": ppf.FAST | ppf.UNFUSED}[a.mode]
    with ppf.Plan(C, T, ppf.generate_prototype(C, T), flags=flags) as p:
        for _ in range(a.reps):
            if a.op == "fir":
                p.fir(x, out=y)
            elif a.op == "fft":
                p.channelize(y, out=y)
            else:
                p.fir_fft(x, out=y)
        torch.cuda.synchronize()
    print("ok", a.op, C, T, S)


if __name__ == "__main__":
    main()
