"""Full-size parity at the BASELINE.json configurations: EVERY output spectrum
of a device-resident run compared with the reference's own CPU implementation
(oracle/_ref: ppf_fir_optimized -> channelize_block, fir.hpp:158-212 and
dft.hpp:175-235, all host cores), the whole-input one-shot being the oracle as
in pipeline_test.cpp:40-51.

  * EXACT (FP64 FIR in the reference order): bit-identical, every output.
  * FAST  (FP32 FIR): max|d| / RMS <= 1e-5 * log2(C) over every output
    (BASELINE.json north_star tolerance).

Sizes: configs[0] (C=512, T=8, 2^17 spectra) in full; the long-stream config
(C=1024, T=16) on a 1 GiB segment; the taps sweep (C=1024, T=4..64) and the
channel sweep (C=64..8192, T=8) at 1 GiB each. The 6.5 GB SKA config is
checked in full by bench.py's `parity` record on every bench run.
"""
import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GIB = 1 << 30


def _ppf():
    from paper_1411_3656_b200 import ppf
    return ppf


def _reference():
    import oracle
    r = oracle.reference()
    if r is None:
        pytest.fail("oracle/_ref (the compiled reference) is missing: run __graft_entry__.build()")
    return r


def _compare(y, want_dev):
    """(max|d|/RMS, outputs whose bits differ) over all outputs, on the GPU."""
    import torch
    w64 = want_dev.to(torch.complex128)
    rms = float((w64.real ** 2 + w64.imag ** 2).mean()) ** 0.5
    d = float((y.to(torch.complex128) - w64).abs().max())
    mism = int((torch.view_as_real(y).view(torch.int32) !=
                torch.view_as_real(want_dev).view(torch.int32)).any(-1).sum())
    return d / rms, mism


CASES = [
    # (id, C, T, S_in)
    ("cfg1", 512, 8, 1 << 17),                        # BASELINE configs[0], in full
    ("long16-1GiB", 1024, 16, GIB // (1024 * 8) + 15),  # configs[4] shape, 1 GiB segment
    ("taps-T4", 1024, 4, GIB // (1024 * 8)),
    ("taps-T32", 1024, 32, GIB // (1024 * 8)),
    ("taps-T64", 1024, 64, GIB // (1024 * 8)),
    ("chan-C64", 64, 8, GIB // (64 * 8)),
    ("chan-C2048", 2048, 8, GIB // (2048 * 8)),
    ("chan-C4096", 4096, 8, GIB // (4096 * 8)),
    ("chan-C8192", 8192, 8, GIB // (8192 * 8)),
]


@pytest.mark.parametrize("name,C,T,S", CASES, ids=[c[0] for c in CASES])
def test_baseline_config_every_output(cuda, name, C, T, S):
    import os
    import torch
    ppf = _ppf()
    ref = _reference()
    x = torch.empty((S, C), dtype=torch.complex64, device=cuda)
    ppf.synth(C, S * C, seed=20141103, out=x)
    coeffs = ref.generate_prototype(C, T)
    S_out = S - T + 1
    torch.cuda.synchronize()
    want = ref.fir_fft(x.cpu().numpy(), C, T, coeffs, workers=os.cpu_count() or 1)
    want_dev = torch.from_numpy(want.view(np.complex64).reshape(S_out, C)).to(cuda)
    with ppf.Plan(C, T, coeffs, flags=ppf.EXACT) as p:
        y = p.fir_fft(x)
        torch.cuda.synchronize()
        err, mism = _compare(y, want_dev)
        assert y.shape == (S_out, C)
        assert mism == 0, f"EXACT ({p.kernel_name}): {mism} of {S_out * C} outputs differ"
        assert err == 0.0
    del y
    with ppf.Plan(C, T, coeffs, flags=ppf.FAST) as p:
        y = p.fir_fft(x)
        torch.cuda.synchronize()
        err, _ = _compare(y, want_dev)
        assert err <= 1e-5 * np.log2(C), f"FAST ({p.kernel_name}): max|d|/RMS {err}"


def test_process_stream_pool_reuse_across_row_sizes(cuda, port):
    """Pooled process_stream buffers reused by a call with the same block bytes
    but twice the row size (C=1024 x 128 spectra, then C=2048 x 64): the reuse
    check must compare byte capacities."""
    ppf = _ppf()
    for C, bs in ((1024, 128), (2048, 64), (1024, 128), (4096, 32)):
        T, S = 8, 700
        src = ppf.synth(C, S * C, seed=C).tobytes()
        coeffs = port.generate_prototype(C, T, 9.0)
        want, st_want = port.process_stream(src, C, T, bs, coeffs)
        sink = io.BytesIO()
        st = ppf.process_stream(C, T, io.BytesIO(src), sink, block_spectra=bs,
                                coefficients=ppf.FilterCoefficients(C, T, coeffs))
        assert sink.getvalue() == want, (C, bs)
        assert st.spectra_processed == st_want.spectra_processed


def test_process_stream_short_reads_are_not_the_end(cuda, port):
    """A source that returns fewer bytes than asked (a pipe) keeps streaming
    until it returns nothing; the output equals the one-shot's bytes."""
    ppf = _ppf()
    C, T, S = 256, 8, 900
    src = ppf.synth(C, S * C, seed=4).tobytes()
    coeffs = port.generate_prototype(C, T, 9.0)
    want, _ = port.process_stream(src, C, T, 64, coeffs)

    class Trickle(io.RawIOBase):
        def __init__(self, data):
            self.data, self.pos, self.k = data, 0, 0

        def read(self, n):
            self.k += 1
            take = min(n, 1 + (self.k * 7919) % (3 * C * 8), len(self.data) - self.pos)
            out = self.data[self.pos:self.pos + take]
            self.pos += take
            return out

    sink = io.BytesIO()
    ppf.process_stream(C, T, Trickle(src), sink, block_spectra=64,
                       coefficients=ppf.FilterCoefficients(C, T, coeffs))
    assert sink.getvalue() == want


def test_multi_device_empty_segment_with_null_buffers(cuda, port):
    """An empty segment may pass null buffers (ppfg.h); it gets 0 outputs."""
    import ctypes as C_
    import torch
    from paper_1411_3656_b200 import _lib
    ppf = _ppf()
    lib = _lib.load()
    C, T = 512, 8
    coeffs = port.generate_prototype(C, T, 9.0)
    rows = [900, 0, 700]
    x = ppf.synth(C, sum(rows) * C, seed=2).reshape(-1, C)
    want = port.fir_fft(x, C, T, coeffs).view(np.complex64).reshape(-1, C)
    plans = [ppf.Plan(C, T, coeffs, flags=ppf.EXACT) for _ in rows]
    segs, outs, o = [], [], 0
    for r in rows:
        if r == 0:
            segs.append(None)
            outs.append(None)
            continue
        t = torch.zeros((r + T - 1, C), dtype=torch.complex64, device=cuda)
        t[:r] = torch.from_numpy(x[o:o + r]).to(cuda)
        segs.append(t)
        outs.append(torch.empty((r, C), dtype=torch.complex64, device=cuda))
        o += r
    torch.cuda.synchronize()
    n = len(rows)
    ph = (_lib.vp * n)(*[p.handle.value for p in plans])
    ins = (_lib.vp * n)(*[t.data_ptr() if t is not None else None for t in segs])
    os_ = (_lib.vp * n)(*[t.data_ptr() if t is not None else None for t in outs])
    got_rows = (_lib.u64 * n)()
    rc = lib.ppfg_multi_fir_fft_device(ph, n, ins, (_lib.u64 * n)(*rows), os_, got_rows)
    assert rc == 0, lib.ppfg_last_error()
    assert list(got_rows) == [900, 0, 700 - T + 1]
    got = np.concatenate([outs[0][:900].cpu().numpy(), outs[2][:700 - T + 1].cpu().numpy()])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    for p in plans:
        p.close()


def test_dropin_stream_exceptions_reach_the_caller(cuda):
    """C++ drop-in process_stream with throwing istream / ostream: the
    exception (or decode_error at the byte offset) reaches the caller, after
    the bytes delivered before the failure were processed (tests/cpp)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "stream_exceptions")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok:") == 3, r.stdout
