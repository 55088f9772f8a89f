#!/usr/bin/env python
"""bench.py — PPF input GB/s, x real-time (6.5 GB/s) and HBM-roofline fraction
on 1..8 B200 (BASELINE.json metric), one process per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config ska|cfg1|...]
                  [--mode fast|exact|unfused] [--impl ours|reference]

A step = one pass of the fused FIR+FFT hot path (ppfg_fir_fft) over one
batch: the whole SKA-LFAA second (C=1024, T=8, 793,457 spectra = 6.5e9 B)
per GPU. With N GPUs every rank takes the next contiguous 6.5 GB segment of
one stream (+ its (T-1)-spectrum halo, generated in place: no communication),
so per-GPU work is fixed ("weak"); value = all ranks' input bytes / the max
over ranks of the device-timed region.

`value`   device-resident (inputs already in HBM), CUDA events on the kernel's
          stream, barrier + synchronize around the K timed steps.
`e2e`     the same metric through the public C-ABI call with HOST buffers
          (pinned): every step copies the input H2D and the spectra D2H inside
          ppfg_fir_fft's chunked double-buffered pipeline.
`roofline` the dominant (only) kernel: algorithmic bytes 8*C*(S_in+S_out) per
          launch / mean launch time vs the measured HBM copy peak.
`exact`   the same step in the reference's own precision (FP64 FIR
          accumulation, bit-identical to ppf_fir_optimized -> channelize_block):
          CUDA-event time, roofline fraction, and a bitwise check of its whole
          output.
`parity`  the WHOLE timed output (every spectrum of rank 0's shard) against the
          reference's CPU implementation (oracle/_ref: ppf_fir_optimized ->
          channelize_block, fir.hpp:158-212 / dft.hpp:175-235, all host cores),
          in chunks: FAST max|d|/RMS (north star bar 1e-5*log2 C), EXACT bitwise.
`cpu_baseline` the reference's own CPU compute pass (oracle/_ref: carry_history
          -> ppf_fir_optimized -> channelize_block, bench.hpp:129-150) on all
          host cores and on one, plus ppf_fir_optimized alone, on bounded
          samples, rank 0 at N=1 only.

The reference arm (--impl reference) loads nothing from paper_1411_3656_b200:
coefficients come from the reference's own generate_prototype and the input
from the oracle's copy of the synthetic generator (oracle/ppf_oracle.c).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PPF input GB/s & ×real-time (6.5 GB/s) vs HBM roofline at 1/2/4/8 B200"
SKA_RATE = 6.5e9                      # bytes/s, pipeline.hpp:17
FALLBACK_HBM_GBS = 6650.0             # /opt/skills/guides/B200_PROFILING.md fallback

CONFIGS = {
    # name: (C, T, S_in per GPU, description)
    "ska": (1024, 8, 793_457, "SKA-LFAA single channel: C=1024, T=8, 793,457 spectra "
                              "(6.5e9 B, 1 s) complex fp32 per GPU"),
    "cfg1": (512, 8, 1 << 17, "PPF C=512, T=8, 2^17 spectra complex fp32"),
    "long16": (1024, 16, 7_812_500, "long stream C=1024, T=16, 64e9 B (sharded)"),
}


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for k, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(C, T, coeffs, sample_spectra, reps, workers):
    """Time the reference's own CPU compute pass (bench.hpp:129-150) on a bounded
    sample of the same workload. Returns (GB/s of input, kind, cores, seconds)."""
    import oracle
    x = oracle.port().synth(C, sample_spectra * C, seed=1)
    ref = oracle.reference()
    if ref is not None:
        secs, emitted = ref.compute_pass(x, C, T, coeffs, block_spectra=4096, workers=workers,
                                         reps=reps + 1)
        secs = secs[1:]  # first rep is the warm-up (bench.hpp:152-153)
        kind, cores = "reference", workers
    else:
        port = oracle.port()
        secs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            port.fir_fft(x, C, T, coeffs)
            secs.append(time.perf_counter() - t0)
        kind, cores = "port", 1
    t = float(np.median(secs))
    return sample_spectra * C * 8 / t / 1e9, kind, cores, secs


def cpu_fir_alone(C, T, coeffs, sample_spectra, reps, workers):
    """ppf_fir_optimized alone (fir.hpp:158-212), one-shot on a bounded sample,
    best of `reps`: GB/s of input."""
    import oracle
    ref = oracle.reference()
    if ref is None:
        return None
    x = oracle.port().synth(C, sample_spectra * C, seed=1)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        ref.fir(x, C, T, coeffs, reference=False, workers=workers)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return sample_spectra * C * 8 / best / 1e9


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path on this
    box's host cores (oracle/_ref), rank 0 only. Nothing of the product
    (paper_1411_3656_b200 / libppfg.so) is loaded on this arm."""
    if rank != 0:
        return
    C, T, S_in, desc = CONFIGS[args.config]
    import oracle
    ref = oracle.reference()
    coeffs = ref.generate_prototype(C, T) if ref is not None else \
        oracle.port().generate_prototype(C, T)           # coeff.hpp:110-144
    workers = os.cpu_count() or 1
    sample = max(T, (args.cpu_sample_mib << 20) // (C * 8))
    x = oracle.port().synth(C, sample * C, seed=1)
    step_times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if ref is not None:
            ref.compute_pass(x, C, T, coeffs, block_spectra=4096, workers=workers, reps=1)
        else:
            oracle.port().fir_fft(x, C, T, coeffs)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            step_times.append(dt)
    kind = "reference" if ref is not None else "port"
    cores = workers if ref is not None else 1
    t = float(np.mean(step_times))
    gbs = sample * C * 8 / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64-acc FIR + f32 FFT (CPU)", "data": "synthetic",
        "x_realtime": gbs * 1e9 / SKA_RATE,
        "config": {"workload": desc, "n_channels": C, "n_taps": T,
                   "sample_spectra": sample, "sample_bytes": sample * C * 8},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} spectra ({sample * C * 8 / 2**20:.0f} MiB) of the "
                                   f"{args.config} workload per step, compute pass with "
                                   f"block_spectra=4096, workers={cores}"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def full_parity(x, outputs, C, T, coeffs, chunk_rows):
    """Compare every output spectrum of the timed run with the reference's CPU
    implementation (oracle/_ref ppf_fir_optimized -> channelize_block, all host
    cores; the oracle port if the reference was not built), chunk by chunk.
    outputs: {"fast": y, "exact": y2, ...} device tensors [S_out, C] complex64.
    Returns {name: {...}} with max|d|/RMS over all outputs and, for exact
    modes, the count of outputs whose bits differ."""
    import torch
    import oracle
    ref = oracle.reference()
    workers = os.cpu_count() or 1
    S_out = next(iter(outputs.values())).shape[0]
    acc = {k: {"maxd": 0.0, "mism": 0} for k in outputs}
    sumsq = 0.0
    t0 = time.perf_counter()
    for o in range(0, S_out, chunk_rows):
        n = min(chunk_rows, S_out - o)
        xin = x[o:o + n + T - 1].cpu().numpy()
        if ref is not None:
            want = ref.fir_fft(xin, C, T, coeffs, workers=workers)
        else:
            want = oracle.port().fir_fft(xin, C, T, coeffs)
        wd = torch.from_numpy(want.view(np.complex64).reshape(n, C)).to(x.device)
        w64 = wd.to(torch.complex128)
        sumsq += float((w64.real ** 2 + w64.imag ** 2).sum())
        for k, y in outputs.items():
            yk = y[o:o + n]
            acc[k]["maxd"] = max(acc[k]["maxd"], float((yk.to(torch.complex128) - w64).abs().max()))
            acc[k]["mism"] += int((torch.view_as_real(yk).view(torch.int32) !=
                                   torch.view_as_real(wd).view(torch.int32)).any(-1).sum())
        del wd, w64
    rms = (sumsq / (S_out * C)) ** 0.5
    out = {}
    for k, a in acc.items():
        out[k] = {"n_outputs": S_out * C, "max_err_over_rms": a["maxd"] / rms if rms else a["maxd"],
                  "outputs_not_bit_identical": a["mism"],
                  "bit_identical": a["mism"] == 0,
                  "tolerance": 1e-5 * float(np.log2(C)) if C > 1 else 1e-6,
                  "checker": ("oracle/_ref (the reference compiled from its sources, "
                              f"ppf_fir_optimized -> channelize_block, workers={workers})")
                  if ref is not None else "oracle port (C restatement, 1 thread)"}
        out[k]["pass"] = bool(out[k]["max_err_over_rms"] <= out[k]["tolerance"])
    out["seconds"] = time.perf_counter() - t0
    return out


def pcie_probe(hx, hy, dx, dy, n_bytes=1 << 30, reps=3):
    """Raw pinned copy bandwidth of this box (GB/s, per direction): H2D alone,
    D2H alone, and both at once — the ceiling the e2e number runs against."""
    import torch

    def raw(t):
        return torch.view_as_real(t).reshape(-1).view(torch.uint8)

    n = min(n_bytes, hx.numel() * 8, hy.numel() * 8, dx.numel() * 8, dy.numel() * 8)
    hi, ho, di, do = raw(hx)[:n], raw(hy)[:n], raw(dx)[:n], raw(dy)[:n]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)

    def both():
        h2d()
        d2h()

    out = {}
    for name, fn in (("h2d", h2d), ("d2h", d2h), ("bidir_each_way", both)):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out[name] = n * reps / (time.perf_counter() - t0) / 1e9
    return out


def ncu_traffic(C, T, mode, n_spectra_in, kernel_name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from a committed `ncu --set full` capture of this same
    configuration AND this same kernel (profiles/*/traffic_*.json, matched on
    the kernel's template configuration); None if there is none."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic_*.json")), reverse=True):
        try:
            t = json.load(open(f))
        except (OSError, ValueError):
            continue
        # "fused_fir_fft_kernel<FusedCfg<...>>" -> "FusedCfg<...>", a substring of
        # ncu's "void fused_fir_fft_kernel<FusedCfg<...>, 0>(...)"
        cfg = kernel_name[kernel_name.find("<") + 1:-1] if "<" in kernel_name else kernel_name
        if (t.get("n_channels"), t.get("n_taps"), t.get("mode"), t.get("n_spectra_in")) == \
                (C, T, mode, n_spectra_in) and cfg and cfg in t.get("kernel", ""):
            return t["traffic_per_launch"], os.path.relpath(f, ROOT)
    return None, None


def time_steps(step, stream, steps):
    """K timed steps on `stream`: (total seconds, mean per-launch seconds)."""
    import torch
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    per = []
    ev0.record(stream)
    for _ in range(steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        per.append((a, b))
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / 1e3, float(np.mean([a.elapsed_time(b) for a, b in per])) / 1e3


def _median_time(fn, reps=5, warm=2):
    """Median device time of one fn() launch, CUDA events on torch's current
    stream (which the library's calls run on), after warm-ups. The reps are
    queued back to back and synchronised once: each launch's events then
    bracket the kernel alone, not the host's submission of the next call (a
    synchronise after every rep would add the ~10 us host path of a library
    call to each 0.3 ms point); the first rep, queued behind an idle GPU, is
    dropped. Inputs are >= 512 MiB (> the 126 MB L2), so no rep finds the
    previous one's data in cache."""
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
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


def config_points(dev, peak, long_bytes):
    """Every BASELINE.json configuration on this GPU, device-resident (the
    SKA headline is the main line): configs[0] cfg1 in full, the taps sweep
    (C=1024, T=4..64) and channels sweep (T=8, C=64..8192) at 1 GiB, and the
    long stream (C=1024, T=16) at `long_bytes` (64e9 = the whole stream on one
    GPU). Per point FAST and EXACT fir_fft, and at each channel count the
    bit-exact FFT alone (channelize_block) beside cuFFT (torch.fft.fft, the
    comparison point, not bit-exact); at each tap count the bit-exact FIR
    alone (ppf_fir_optimized); detection (fused mean power) at
    C=1024 T=8. Median of 5 after 2 warm-ups; frac = (in + out) / t / peak
    (detection: in / t / peak, the fused pass being read-only)."""
    import torch
    from paper_1411_3656_b200 import ppf
    pts = [("cfg1", 512, 8, 1 << 17)]
    pts += [("taps", 1024, t, (1 << 30) // (1024 * 8)) for t in (4, 8, 16, 32, 64)]
    pts += [("channels", c, 8, (1 << 30) // (c * 8)) for c in (64, 128, 256, 512, 1024, 2048, 4096, 8192)]
    if long_bytes:
        pts.append(("long16", 1024, 16, long_bytes // (1024 * 8)))
    out = []
    for name, C, T, S in pts:
        try:
            x = torch.empty((S, C), dtype=torch.complex64, device=dev)
            y = torch.empty((S - T + 1, C), dtype=torch.complex64, device=dev)
        except RuntimeError as e:  # out of memory: report, keep going
            out.append({"config": name, "C": C, "T": T, "S_in": S, "error": str(e)[:120]})
            torch.cuda.empty_cache()
            continue
        ppf.synth(C, S * C, seed=3, out=x)
        coeffs = ppf.generate_prototype(C, T)
        bi, bo = S * C * 8, (S - T + 1) * C * 8
        r = {"config": name, "C": C, "T": T, "S_in": S, "bytes_in": bi}
        for mode, flags in (("fast", ppf.FAST), ("exact", ppf.EXACT)):
            with ppf.Plan(C, T, coeffs, flags=flags) as p:
                t = _median_time(lambda: p.fir_fft(x, out=y))
                r[mode] = {"ms": t * 1e3, "input_gbps": bi / t / 1e9,
                           "x_realtime": bi / t / SKA_RATE, "frac": (bi + bo) / t / 1e9 / peak,
                           "kernel": p.kernel_name}
        if name == "channels":
            with ppf.Plan(C, 0) as p:
                t = _median_time(lambda: p.channelize(y, out=y))
            tc = _median_time(lambda: torch.fft.fft(y, dim=1))
            r["fft_only"] = {"ms": t * 1e3, "frac": 2 * bo / t / 1e9 / peak,
                             "what": "channelize_block, bit-exact radix-2, in place"}
            r["cufft"] = {"ms": tc * 1e3, "frac": 2 * bo / tc / 1e9 / peak,
                          "what": "torch.fft.fft (cuFFT), comparison only, not bit-exact"}
        if name == "taps":  # the FIR alone (ppf_fir_optimized, bit-exact)
            with ppf.Plan(C, T, coeffs) as p:
                t = _median_time(lambda: p.fir(x, out=y))
            r["fir_only"] = {"ms": t * 1e3, "frac": (bi + bo) / t / 1e9 / peak,
                             "what": "ppf_fir_optimized (fir.hpp:158-212), bit-exact"}
        if name == "taps" and T == 8:
            with ppf.Plan(C, T, coeffs, flags=ppf.FAST) as p:
                t = _median_time(lambda: p.fir_fft_mean_power(x))
            r["detect"] = {"ms": t * 1e3, "input_gbps": bi / t / 1e9, "frac_read_only": bi / t / 1e9 / peak,
                           "what": "fir_fft_mean_power (cmd_inspect, cli.hpp:307-317), FAST"}
        out.append(r)
        del x, y
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="ska", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="fast", choices=["fast", "exact", "unfused"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-mib", type=int, default=1024)
    ap.add_argument("--spectra", type=int, default=0, help="override S_in per GPU")
    ap.add_argument("--no-exact", action="store_true", help="skip the EXACT-mode sub-record")
    ap.add_argument("--no-parity", action="store_true", help="skip the whole-output check")
    ap.add_argument("--parity-chunk-mib", type=int, default=512)
    ap.add_argument("--parity-all-ranks", action="store_true",
                    help="every rank checks its own shard (default: rank 0 only)")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE config sweep")
    ap.add_argument("--long-gb", type=float, default=64.0,
                    help="long-stream config size on one GPU (GB of input; 0 = skip)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    # test mode (tests/test_gpu_multirank.py): every rank on one device with
    # gloo for the barrier / max-over-ranks, so the rank path (shards, halos,
    # timing reduction) runs on real kernels on a one-GPU box
    backend = os.environ.get("PPFG_BENCH_BACKEND", "nccl")
    if os.environ.get("PPFG_BENCH_SAME_DEVICE"):
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local_rank)
    from paper_1411_3656_b200 import ppf

    C, T, S_per, desc = CONFIGS[args.config]
    if args.spectra:
        S_per = args.spectra
    if args.config == "long16":
        # the 64e9-byte stream is SHARDED across ranks (strong scaling)
        S_total = S_per
        ib, ic, ob, oc = ppf.shard_range(S_total, T, rank, world)
        scaling = "strong"
    else:
        # every rank its own contiguous S_per-spectrum segment of one stream
        S_total = S_per * world + T - 1
        ib, ic, ob, oc = ppf.shard_range(S_total, T, rank, world)
        scaling = "weak"
    flags = {"fast": ppf.FAST, "exact": ppf.EXACT, "unfused": ppf.UNFUSED}[args.mode]
    coeffs = ppf.generate_prototype(C, T)
    plan = ppf.Plan(C, T, coeffs, flags=flags, device=local_rank)
    stream = torch.cuda.current_stream(dev)

    x = torch.empty((ic, C), dtype=torch.complex64, device=dev)
    y = torch.empty((oc, C), dtype=torch.complex64, device=dev)
    ppf.synth(C, ic * C, seed=1, first_sample=ib * C, out=x)   # the shard + its halo, in place
    torch.cuda.synchronize()

    bytes_in = ic * C * 8          # per rank, halo included (it is read)
    bytes_out = oc * C * 8
    alg_bytes = bytes_in + bytes_out

    def step():
        plan.fir_fft(x, out=y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    launches0 = ppf.kernel_launches()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_total, t_launch = time_steps(step, stream, args.steps)
    if world > 1:
        dist.barrier()
    launches = ppf.kernel_launches() - launches0
    clocks = sampler.stop()
    t_max = max_over_ranks(t_total)
    in_all = sum_over_ranks(bytes_in)
    value = in_all * args.steps / t_max / 1e9

    peak, peak_src = measured_peak()
    achieved = alg_bytes / t_launch / 1e9

    # ---- the same step in the reference's precision (EXACT, bit-identical) ----
    exact = None
    y_exact = None
    if args.mode == "fast" and not args.no_exact:
        with ppf.Plan(C, T, coeffs, flags=ppf.EXACT, device=local_rank) as pe:
            y_exact = torch.empty((oc, C), dtype=torch.complex64, device=dev)

            def step_exact():
                pe.fir_fft(x, out=y_exact)

            for _ in range(args.warmup):
                step_exact()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            te_total, te_launch = time_steps(step_exact, stream, args.steps)
            te_max = max_over_ranks(te_total)
            v_exact = in_all * args.steps / te_max / 1e9
            exact = {"value": v_exact, "unit": "GB/s", "x_realtime": v_exact * 1e9 / SKA_RATE,
                     "ms_per_step": te_max / args.steps * 1e3,
                     "dtype": "f64-acc FIR + f32 FFT (reference order)",
                     "kernel": pe.kernel_name,
                     "roofline": {"bound": "hbm", "achieved": alg_bytes / te_launch / 1e9,
                                  "peak": peak, "unit": "GB/s",
                                  "frac": alg_bytes / te_launch / 1e9 / peak,
                                  "launch_ms": te_launch * 1e3}}
            tr, tr_src = ncu_traffic(C, T, "exact", ic, pe.kernel_name)
            exact["roofline"]["traffic"] = tr
            exact["roofline"]["traffic_source"] = tr_src

    # ---- parity: every output spectrum of the timed runs vs the reference ----
    parity = None
    if args.parity_all_ranks and not args.no_parity:
        # every rank checks its own shard (halo included) and the worst one is
        # reported: max err over ranks, mismatch counts summed
        chunk = max(1, (args.parity_chunk_mib << 20) // (C * 8))
        mine = full_parity(x, {args.mode: y}, C, T, coeffs.values, chunk)[args.mode]
        parity = {args.mode: dict(mine, ranks=world,
                                  max_err_over_rms=max_over_ranks(mine["max_err_over_rms"]),
                                  outputs_not_bit_identical=int(sum_over_ranks(
                                      mine["outputs_not_bit_identical"])),
                                  n_outputs=int(sum_over_ranks(mine["n_outputs"]))),
                  "seconds": None}
        p = parity[args.mode]
        p["bit_identical"] = p["outputs_not_bit_identical"] == 0
        p["pass"] = bool(p["max_err_over_rms"] <= p["tolerance"])
    elif rank == 0 and not args.no_parity:
        outs = {args.mode: y}
        if y_exact is not None:
            outs["exact"] = y_exact
        chunk = max(1, (args.parity_chunk_mib << 20) // (C * 8))
        parity = full_parity(x, outs, C, T, coeffs.values, chunk)
        if exact is not None:
            exact["parity"] = parity.pop("exact")
    del y_exact

    # ---- end to end through the public C-ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        hx = torch.empty((ic, C), dtype=torch.complex64, pin_memory=True)
        hy = torch.empty((oc, C), dtype=torch.complex64, pin_memory=True)
        hx.copy_(x)
        torch.cuda.synchronize()
        plan.fir_fft(hx, out=hy)  # warm-up (allocates the pipeline buffers)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.fir_fft(hx, out=hy)
            _ = float(hy[-1, 0].real)   # host read of the step's result
        te = time.perf_counter() - t0
        te_max = max_over_ranks(te)
        row_b = C * 8
        chunk = max(1, min(oc, (64 << 20) // row_b))
        n_chunks = -(-oc // chunk)
        h2d = (oc + n_chunks * (T - 1)) * row_b
        e2e = {"value": in_all * args.e2e_steps / te_max / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(oc * row_b),
               "steps": args.e2e_steps, "x_realtime": in_all * args.e2e_steps / te_max / SKA_RATE,
               "path": "ppfg_fir_fft(mem=HOST), pinned buffers, 64 MiB double-buffered chunks",
               "pcie_limit": pcie_probe(hx, hy, x, y)}
        # the same call with pageable host buffers (what a reference caller
        # holds): staged through pinned memory by the library's copy threads
        # (one rank only: N ranks x 13 GB more host memory otherwise)
        if world > 1:
            del hx, hy
    if e2e is not None and world == 1:
        px = hx.numpy().copy()
        py = np.empty((oc, C), np.complex64)
        del hx, hy
        plan.fir_fft(px, out=py)      # warm-up (staging buffers, page faults of py)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.fir_fft(px, out=py)
            _ = float(py[-1, 0].real)
        tp = max_over_ranks(time.perf_counter() - t0)
        e2e["pageable"] = {"value": in_all * args.e2e_steps / tp / 1e9, "unit": "GB/s",
                           "x_realtime": in_all * args.e2e_steps / tp / SKA_RATE,
                           "path": "ppfg_fir_fft(mem=HOST), pageable numpy buffers, staged through "
                                   "pinned memory by the copy threads in 8 MiB chunks"}
        del px, py

    # ---- CPU baseline: the reference on this host, N=1 rank 0 only ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        sample = max(T, (args.cpu_sample_mib << 20) // (C * 8))
        gbs, kind, cores, secs = cpu_reference_sample(C, T, coeffs.values, sample, 2, workers)
        sample1 = max(T, (args.cpu_sample_mib << 20) // 4 // (C * 8))
        gbs1, _, cores1, secs1 = cpu_reference_sample(C, T, coeffs.values, sample1, 1, 1)
        fir_gbs = cpu_fir_alone(C, T, coeffs.values, sample, 3, workers)
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind,
               "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
               "sample": f"{sample} spectra ({sample * C * 8 / 2**20:.0f} MiB) of the same "
                         f"workload, reference compute pass (bench.hpp:129-150), "
                         f"block_spectra=4096, median of {len(secs)}",
               "x_realtime": gbs * 1e9 / SKA_RATE,
               "single_core": {"value": gbs1, "unit": "GB/s", "cores": cores1,
                               "sample": f"{sample1} spectra, same compute pass, workers=1"},
               "fir_alone": {"value": fir_gbs, "unit": "GB/s", "cores": workers,
                             "sample": f"{sample} spectra, ppf_fir_optimized one-shot "
                                       f"(fir.hpp:158-212), best of 3"}}

    # ---- every BASELINE.json configuration (N=1 rank 0): the sweeps ----
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        del x, y
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        configs = {"points": config_points(dev, peak, int(args.long_gb * 1e9)),
                   "peak_gbps": peak, "seconds": None,
                   "timing": "median of 5 back-to-back launches after 2 warm-ups, CUDA events, device-resident; "
                             "1 GiB points, cfg1 and long16 at their full size"}
        configs["seconds"] = time.perf_counter() - t0

    if rank == 0:
        kind = plan.kind
        kname = plan.kernel_name
        traffic, traffic_src = ncu_traffic(C, T, args.mode, ic, kname)
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None,
            "dtype": {"fast": "f32", "exact": "f64-acc FIR + f32 FFT",
                      "unfused": "f64-acc FIR + f32 FFT"}[args.mode],
            "data": "synthetic (counter-based tone+noise, generated on device per shard)",
            "x_realtime": value * 1e9 / SKA_RATE,
            "config": {"workload": desc, "n_channels": C, "n_taps": T,
                       "n_spectra_in_per_gpu": ic, "bytes_in_per_gpu": bytes_in,
                       "mode": args.mode, "kernel": ["unfused", "fused-fp32", "fused-fp64", "cluster-fp32", "cluster-fp64", "tiny-fp32", "tiny-fp64", "l2x-fp32", "l2x-fp64"][kind],
                       "l2": "inputs >> 126 MB L2 (no flush needed)", "parallelism": f"shard{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": alg_bytes,
                         "launch_ms": t_launch * 1e3, "kernel": kname,
                         "traffic_source": traffic_src},
            "parity": parity.get(args.mode) if parity else None,
            "exact": exact,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "configs": configs,
            "clocks": clocks,
            "gpu_launches": int(launches),
        }
        if parity:
            line["parity"]["seconds"] = parity["seconds"]
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
