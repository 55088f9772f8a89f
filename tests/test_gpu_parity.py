"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same
seeded inputs and against the reference's golden vectors.

Bars (SURVEY §8c / BASELINE.json north_star):
  * FIR (K1), FFT (K2), dft_naive (K4), fused EXACT (K3 fp64) and streaming:
    bit-identical to the reference.
  * fused FAST (K3 fp32 FIR): max|err|/RMS <= 1e-5 * log2(C) (north star).
"""
import io

import numpy as np
import pytest

from conftest import bits, max_err_over_rms, uniform

pytestmark = pytest.mark.gpu


def ppf_mod():
    from paper_1411_3656_b200 import ppf
    return ppf


# ---------------------------------------------------------------- FIR (K1)
def test_fir_golden_bitwise(cuda, golden):
    ppf = ppf_mod()
    for i in range(int(golden["n_fir"])):
        C, T = int(golden[f"fir{i}_C"]), int(golden[f"fir{i}_T"])
        x, c = golden[f"fir{i}_x"].view(np.complex64), golden[f"fir{i}_coeffs"]
        with ppf.Plan(C, T, c) as p:
            assert np.array_equal(bits(p.fir(x)), bits(golden[f"fir{i}_y"])), (C, T)
            assert np.array_equal(bits(p.fir_reference(x)), bits(golden[f"fir{i}_y_ref"])), (C, T)


@pytest.mark.parametrize("C", [1, 2, 3, 8, 64, 100, 256, 1024, 4096])
@pytest.mark.parametrize("T", [1, 2, 4, 7, 8, 12, 16, 17, 20, 24, 32, 48, 64, 128])
def test_fir_bitwise_vs_oracle(cuda, port, C, T):
    ppf = ppf_mod()
    rng = np.random.default_rng(C * 1000 + T)
    S = T + int(rng.integers(0, 40)) + (3000 if C <= 64 else 0)
    x = uniform(rng, S * C)
    coeffs = port.generate_prototype(C, T, 9.0)
    with ppf.Plan(C, T, coeffs) as p:
        got = p.fir(x)
    with ppf.Plan(C, T, coeffs, flags=ppf.K1_PREFETCH) as p:
        got_prefetch = p.fir(x)
    assert got.shape == (S - T + 1, C)
    want = bits(port.fir(x, C, T, coeffs))
    assert np.array_equal(bits(got), want)
    assert np.array_equal(bits(got_prefetch), want)


# K1b (register-blocked FIR, T >= 16): long enough streams for many steps,
# several time segments and ring wrap-arounds, ragged channel counts (partial
# 32-channel blocks), both operation orders; bitwise against the oracle and
# against the lane-window kernels it replaces.
@pytest.mark.parametrize("C,T,S", [(1024, 16, 9000), (1024, 32, 9000), (1024, 64, 9000),
                                   (66, 32, 40000), (1000, 64, 5000), (2, 16, 70000),
                                   (4096, 32, 1500), (128, 64, 64), (96, 16, 16)])
def test_fir_block_bitwise(cuda, port, C, T, S):
    ppf = ppf_mod()
    x = ppf.synth(C, S * C, seed=C + 7 * T)
    coeffs = port.generate_prototype(C, T, 9.0)
    with ppf.Plan(C, T, coeffs) as p:
        got = p.fir(x)
        got_ref = p.fir_reference(x)
    with ppf.Plan(C, T, coeffs, flags=ppf.FIR_LEGACY) as p:
        legacy = p.fir(x)
    want = bits(port.fir(x, C, T, coeffs))
    assert np.array_equal(bits(got), want)
    assert np.array_equal(bits(legacy), want)
    assert np.array_equal(bits(got_ref), bits(port.fir(x, C, T, coeffs, reference_order=True)))


# K1b in FP32 (PPFG_FAST unfused path, T = 32..128): FIR+FFT within the
# north-star bound, and the FP32 FIR alone close to the exact one.
@pytest.mark.parametrize("C,T,S", [(1024, 32, 6000), (1024, 64, 6000), (1024, 128, 3000),
                                   (2048, 64, 1200), (66, 64, 9000)])
def test_fir_block_fast(cuda, port, C, T, S):
    ppf = ppf_mod()
    x = ppf.synth(C, S * C, seed=C * 3 + T)
    coeffs = port.generate_prototype(C, T, 9.0)
    with ppf.Plan(C, T, coeffs, flags=ppf.FAST | ppf.UNFUSED) as p:
        got = p.fir_fft(x)
    want = port.fir_fft(x, C, T, coeffs).view(np.complex64)   # dft_naive for C = 66
    assert max_err_over_rms(got, want) <= 1e-5 * np.log2(C)


def test_fir_errors(cuda):
    ppf = ppf_mod()
    rng = np.random.default_rng(113)
    c = ppf.generate_prototype(8, 4)
    with pytest.raises(ppf.insufficient_history_error):   # fir_test.cpp:129-134
        ppf.ppf_fir_reference(uniform(rng, 8 * 3), c)
    with pytest.raises(ppf.config_error):                 # fir_test.cpp:122-127
        ppf.ppf_fir_optimized(uniform(rng, 8 * 16), ppf.generate_prototype(16, 4), n_channels=8)
    with pytest.raises(ppf.config_error):
        ppf.ppf_fir_optimized(uniform(rng, 8 * 16), c, workers=0)


def test_fir_properties(cuda):
    """fir_test.cpp:171-257: shift equivariance and channel independence are exact;
    a finite impulse response touches exactly T spectra of one channel."""
    ppf = ppf_mod()
    rng = np.random.default_rng(149)
    C, T, S = 8, 4, 24
    c = ppf.generate_prototype(C, T)
    x = uniform(rng, S * C)
    base = ppf.ppf_fir_optimized(x, c)
    moved = ppf.ppf_fir_optimized(np.concatenate([uniform(rng, C), x]), c)
    assert np.array_equal(bits(moved[1:]), bits(base))
    masked = x.copy().reshape(S, C)
    masked[:, 3] = 0
    got = ppf.ppf_fir_optimized(masked, c)
    assert np.all(got[:, 3] == 0)
    keep = [k for k in range(C) if k != 3]
    assert np.array_equal(bits(got[:, keep]), bits(base[:, keep]))
    imp = np.zeros((30, 8), np.complex64)
    imp[14, 5] = 0.5 - 2.0j
    coeffs = ppf.FilterCoefficients(8, 6, rng.uniform(0.25, 1.75, 48))
    y = ppf.ppf_fir_optimized(imp, coeffs)
    nz = y != 0
    assert nz[:, [k for k in range(8) if k != 5]].sum() == 0 and nz[:, 5].sum() == 6


# ---------------------------------------------------------------- FFT (K2/K4)
def test_fft_golden_bitwise(cuda, golden):
    ppf = ppf_mod()
    for n in golden["fft_sizes"]:
        n = int(n)
        got = ppf.channelize_block(golden[f"fft{n}_x"].view(np.complex64), n)
        assert np.array_equal(bits(got), bits(golden[f"fft{n}_y"])), n
    for n in golden["dft_sizes"]:
        n = int(n)
        got = ppf.channelize_block(golden[f"dft{n}_x"].view(np.complex64), n)
        assert np.array_equal(bits(got), bits(golden[f"dft{n}_y"])), n


@pytest.mark.parametrize("L", list(range(0, 17)))
def test_fft_bitwise_vs_oracle(cuda, port, L):
    ppf = ppf_mod()
    n = 1 << L
    rng = np.random.default_rng(L)
    rows = max(3, (1 << 16) // n) + 1
    x = uniform(rng, rows * n)
    got = ppf.channelize_block(x, n)
    assert np.array_equal(bits(got), bits(port.channelize(x, n)))


# C = 8192 channelize (K2n, one 64 KB row per CTA, twiddles of the last pass
# from global): ragged row counts, in place and out of place.
@pytest.mark.parametrize("rows", [1, 2, 149, 700])
def test_fft_ring_many_rows(cuda, port, rows):
    import torch
    ppf = ppf_mod()
    n = 8192
    rng = np.random.default_rng(rows)
    x = uniform(rng, rows * n)
    want = bits(port.channelize(x, n))
    assert np.array_equal(bits(ppf.channelize_block(x, n)), want)
    xd = torch.from_numpy(x.view(np.complex64).reshape(rows, n)).cuda()
    with ppf.Plan(n, 0) as p:
        p.channelize(xd, out=xd)   # in place
    torch.cuda.synchronize()
    assert np.array_equal(bits(xd.cpu().numpy()), want)


def test_fft_api_semantics(cuda, port):
    """dft_test.cpp:72-123, 125-197."""
    ppf = ppf_mod()
    assert ppf.fft(np.array([0.25 - 1.5j], np.complex64))[0] == np.complex64(0.25 - 1.5j)
    d = np.zeros(8, np.complex64)
    d[0] = 1
    assert np.allclose(ppf.fft(d), 1.0)
    with pytest.raises(ppf.unsupported_size_error):
        ppf.fft(np.ones(12, np.complex64))
    x = uniform(np.random.default_rng(241), 6 * 4)
    with pytest.raises(ppf.unsupported_size_error):
        ppf.channelize_block(x, 6, fft_fallback=False)
    assert ppf.channelize_block(np.zeros(0, np.complex64), 4).size == 0
    for n in (3, 12, 100):
        x = uniform(np.random.default_rng(n), n)
        assert np.array_equal(bits(ppf.dft_naive(x)), bits(port.dft_naive(x)))
    for n in (1, 2, 64, 512):
        x = uniform(np.random.default_rng(n), n)
        assert np.array_equal(bits(ppf.fft(x)), bits(port.fft(x)))


def test_channelize_in_place_device(cuda, port):
    import torch
    ppf = ppf_mod()
    for n, rows in ((6, 17), (64, 17), (1024, 17), (2048, 301), (4096, 17), (4096, 733),
                    (8192, 611), (32768, 17)):
        rng = np.random.default_rng(n + rows)
        x = uniform(rng, rows * n)
        t = torch.from_numpy(x.copy()).to(cuda)
        with ppf.Plan(n) as p:
            p.channelize(t, out=t)
        torch.cuda.synchronize()
        assert np.array_equal(bits(t.cpu().numpy()), bits(port.channelize(x, n))), n


# ---------------------------------------------------------------- fused (K3)
def test_fused_golden_exact(cuda, golden):
    ppf = ppf_mod()
    for i in range(int(golden["n_ff"])):
        C, T = int(golden[f"ff{i}_C"]), int(golden[f"ff{i}_T"])
        with ppf.Plan(C, T, golden[f"ff{i}_coeffs"], flags=ppf.EXACT) as p:
            got = p.fir_fft(golden[f"ff{i}_x"].view(np.complex64))
        assert np.array_equal(bits(got), bits(golden[f"ff{i}_y"])), (C, T)


@pytest.mark.parametrize("C,T", [(512, 8), (1024, 8), (64, 8), (256, 4), (2048, 8), (8192, 8), (4096, 8), (1024, 32),
                                 (1024, 4), (1024, 16), (512, 16), (128, 8), (1024, 64), (256, 128),
                                 (256, 8), (64, 4), (128, 16), (256, 16), (64, 16), (512, 4), (128, 4), (256, 32),
                                 (64, 32)])
@pytest.mark.parametrize("flags", ["exact", "fast", "exact+cluster", "fast+cluster", "fast+unfused"])
def test_fused_vs_oracle(cuda, port, C, T, flags):
    ppf = ppf_mod()
    rng = np.random.default_rng(C + T)
    S = T - 1 + 148 * 8 * 3 + int(rng.integers(0, 50))   # several batches per CTA + ragged tail
    if C >= 2048:
        S = T - 1 + 700
    x = ppf.synth(C, S * C, seed=C * 31 + T)
    coeffs = port.generate_prototype(C, T, 9.0)
    want = port.fir_fft(x, C, T, coeffs).view(np.complex64)
    f = (ppf.EXACT if flags.startswith("exact") else ppf.FAST) | \
        (ppf.CLUSTER if flags.endswith("cluster") else 0) | \
        (ppf.UNFUSED if flags.endswith("unfused") else 0)
    with ppf.Plan(C, T, coeffs, flags=f) as p:
        got = p.fir_fft(x)
        kind = p.kind
    assert got.shape == (S - T + 1, C)
    if flags.startswith("exact") or (kind == 0 and T < 16):
        assert np.array_equal(bits(got), bits(want)), f"kind={kind}"
    else:   # FP32 FIR (fused kernels, or K1b FP32 on the FAST unfused path)
        err = max_err_over_rms(got, want)
        assert err <= 1e-5 * np.log2(C), err


@pytest.mark.parametrize("C", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("T", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_tiny_c_fused_vs_oracle(cuda, port, C, T, mode):
    """K6 (tiny.cuh): warp-level fused FIR + shuffle FFT for C = 2..32 —
    EXACT bit-identical, FAST within the north-star bar; ragged segment
    tails, a single output spectrum and a segment count that leaves idle
    lane groups."""
    ppf = ppf_mod()
    coeffs = port.generate_prototype(C, T, 9.0)
    flags = ppf.EXACT if mode == "exact" else ppf.FAST
    for S in (T, T + 1, T + 37, 20000 + T + 3):
        x = ppf.synth(C, S * C, seed=S + C)
        want = port.fir_fft(x, C, T, coeffs).view(np.complex64)
        with ppf.Plan(C, T, coeffs, flags=flags) as p:
            got = p.fir_fft(x)
            kind = p.kind
        assert got.shape == (S - T + 1, C)
        if mode == "exact" or C == 1:   # C = 1 (FIR alone) always runs the FP64 FIR
            assert np.array_equal(bits(got), bits(want)), (S, kind)
        else:
            assert max_err_over_rms(got, want) <= 1e-5 * np.log2(C), (S, kind)
        if not ((mode == "exact" or C == 1) and T == 32):
            assert kind == (6 if (mode == "exact" or C == 1) else 5)


@pytest.mark.parametrize("C,T,mode", [(1024, 32, "fast"), (1024, 64, "fast"), (1024, 16, "fast"),
                                      (1024, 32, "exact"), (8192, 8, "fast"), (8192, 8, "exact")])
def test_l2x_fused_vs_oracle(cuda, port, C, T, mode):
    """K7 (l2x.cuh): FIR -> L2-resident exchange ring -> FFT in one persistent
    kernel. EXACT bit-identical, FAST within the north-star bar; a single
    output, chunk-ragged tails, a multi-round run (more work items than SMs),
    and repeated launches on one plan (the ring and counters are reused)."""
    ppf = ppf_mod()
    coeffs = port.generate_prototype(C, T, 9.0)
    flags = (ppf.EXACT if mode == "exact" else ppf.FAST) | ppf.L2X
    sizes = (T, T + 300, T + 4000) if C == 8192 else (T, T + 255, T + 256, T + 3 * 256 * 148 // 32 + 17)
    with ppf.Plan(C, T, coeffs, flags=flags) as p:
        assert p.kind == (8 if mode == "exact" else 7), p.kernel_name
        for S in sizes:
            x = ppf.synth(C, S * C, seed=S + T)
            want = port.fir_fft(x, C, T, coeffs).view(np.complex64)
            for rep in range(2):
                got = p.fir_fft(x)
                assert got.shape == (S - T + 1, C)
                if mode == "exact":
                    assert np.array_equal(bits(got), bits(want)), (S, rep)
                else:
                    assert max_err_over_rms(got, want) <= 1e-5 * np.log2(C), (S, rep)


@pytest.mark.parametrize("S_extra", [0, 1, 2, 7, 8, 9, 100])
def test_fused_small_and_ragged(cuda, port, S_extra):
    """n_spectra_out = 1 and tails that do not fill a batch (SURVEY §7 hard part 7)."""
    ppf = ppf_mod()
    for C, T, flags in [(512, 8, ppf.EXACT), (1024, 8, ppf.FAST), (512, 8, ppf.FAST),
                        (1024, 16, ppf.FAST | ppf.CLUSTER), (1024, 8, ppf.EXACT | ppf.CLUSTER),
                        (2048, 8, ppf.FAST | ppf.CLUSTER), (8192, 8, ppf.FAST | ppf.CLUSTER)]:
        S = T + S_extra
        x = uniform(np.random.default_rng(S_extra), S * C)
        coeffs = port.generate_prototype(C, T, 9.0)
        want = port.fir_fft(x, C, T, coeffs)
        with ppf.Plan(C, T, coeffs, flags=flags) as p:
            got = p.fir_fft(x)
        if not flags & ppf.FAST:
            assert np.array_equal(bits(got), bits(want)), (C, T, S_extra)
        else:
            assert max_err_over_rms(got, want) <= 1e-5 * np.log2(C)


def test_fused_device_resident_torch(cuda, port):
    import torch
    ppf = ppf_mod()
    C, T, S = 1024, 8, 5000
    with ppf.Plan(C, T, port.generate_prototype(C, T, 9.0), flags=ppf.FAST) as p:
        x = torch.empty((S, C), dtype=torch.complex64, device=cuda)
        ppf.synth(C, S * C, seed=5, out=x)
        y = p.fir_fft(x)
        torch.cuda.synchronize()
        host = ppf.synth(C, S * C, seed=5)
        assert np.array_equal(bits(x.cpu().numpy()), bits(host))   # device == host generator
        want = port.fir_fft(host, C, T, port.generate_prototype(C, T, 9.0))
        assert max_err_over_rms(y.cpu().numpy(), want) <= 1e-5 * np.log2(C)


def test_unfused_flag_is_bitwise_exact(cuda, port):
    ppf = ppf_mod()
    C, T, S = 1024, 8, 3000
    x = ppf.synth(C, S * C, seed=9)
    c = port.generate_prototype(C, T, 9.0)
    with ppf.Plan(C, T, c, flags=ppf.UNFUSED) as p:
        assert p.kind == 0
        assert np.array_equal(bits(p.fir_fft(x)), bits(port.fir_fft(x, C, T, c)))


# ---------------------------------------------------------------- streaming
def test_stream_golden_and_block_invariance(cuda, golden, port):
    """pipeline_test.cpp:156-170 and acceptance criterion 6: byte-identical
    output for any block size, equal to the reference's bytes."""
    ppf = ppf_mod()
    src = golden["stream_x"].tobytes()
    for bs in (8, 100, 999, 4096):
        sink = io.BytesIO()
        st = ppf.process_stream(8, 8, io.BytesIO(src), sink, block_spectra=bs)
        assert sink.getvalue() == golden["stream_y"].tobytes(), bs
        assert [st.spectra_processed, st.bytes_in, st.bytes_out, st.dropped_samples] == \
            [int(v) for v in golden["stream_state"]]
    sink = io.BytesIO()
    ppf.process_stream(8, 8, io.BytesIO(src), sink, block_spectra=64, zero_prime=True)
    assert sink.getvalue() == golden["stream_zp_y"].tobytes()


def test_stream_arbitrary_pushes_equal_one_shot(cuda, port):
    ppf = ppf_mod()
    C, T = 1024, 8
    rng = np.random.default_rng(20140606)
    x = ppf.synth(C, 3000 * C, seed=11)
    raw = x.tobytes()
    coeffs = ppf.generate_prototype(C, T)
    want = port.fir_fft(x, C, T, coeffs.values).tobytes()
    for flags in (ppf.EXACT, ppf.FAST):
        with ppf.Plan(C, T, coeffs, flags=flags) as p:
            s = ppf.Stream(p, block_spectra=512)
            out = b""
            pos = 0
            while pos < len(raw):
                n = int(rng.integers(1, 3 * 8 * C))
                out += s.push(raw[pos:pos + n])
                pos += n
            st = s.close()
            s.destroy()
        assert st.spectra_processed == 3000 - T + 1
        if flags == ppf.EXACT:
            assert out == want
        else:
            assert max_err_over_rms(np.frombuffer(out, np.complex64),
                                    np.frombuffer(want, np.complex64)) <= 1e-5 * np.log2(C)


def test_stream_errors(cuda):
    ppf = ppf_mod()
    rng = np.random.default_rng(349)
    raw = uniform(rng, 4 * 6).tobytes() + b"\x01\x02\x03"
    with pytest.raises(ppf.decode_error) as e:       # pipeline_test.cpp:219-233
        ppf.process_stream(4, 2, io.BytesIO(raw), io.BytesIO(), block_spectra=4)
    assert e.value.byte_offset == 6 * 4 * 8

    class Failing:
        def write(self, b):
            raise OSError("full")
    with pytest.raises(ppf.io_error):                 # pipeline_test.cpp:251-258
        ppf.process_stream(4, 2, io.BytesIO(uniform(rng, 32).tobytes()), Failing(),
                           block_spectra=4)
    with pytest.raises(ppf.config_error):             # pipeline_test.cpp:270-276
        ppf.process_stream(8, 4, io.BytesIO(b""), io.BytesIO(), block_spectra=2)
    st = ppf.process_stream(4, 3, io.BytesIO(uniform(rng, 8).tobytes()), io.BytesIO(),
                            block_spectra=16)
    assert st.spectra_processed == 0                  # pipeline_test.cpp:138-145


# ---------------------------------------------------------------- shards / synth
def test_shards_reassemble_the_one_shot(cuda, port):
    """each shard = its segment + (T-1) halo, no collective; the
    concatenated shard outputs equal the one-shot output bit for bit."""
    ppf = ppf_mod()
    C, T, S = 1024, 16, 4000
    x = ppf.synth(C, S * C, seed=2).reshape(S, C)
    c = ppf.generate_prototype(C, T)
    want = port.fir_fft(x, C, T, c.values).view(np.complex64).reshape(-1, C)
    for world in (1, 2, 3, 8):
        parts = []
        with ppf.Plan(C, T, c) as p:
            for r in range(world):
                ib, ic, ob, oc = ppf.shard_range(S, T, r, world)
                parts.append(p.fir_fft(x[ib:ib + ic]))
        assert np.array_equal(bits(np.concatenate(parts)), bits(want))
    got = ppf.multi_fir_fft(x, c, devices=[0, 0])
    assert np.array_equal(bits(got), bits(want))


# SURVEY §8e halo "from the peer": device segments with spare rows, halos
# copied from the following segment(s) (cudaMemcpyPeerAsync; on one GPU every
# segment shares cuda:0, so the copy path is exercised, not NVLink), outputs
# byte-identical to one ppfg_fir_fft over the stream — including segments
# shorter than the halo and an empty one.
@pytest.mark.parametrize("flags", ["exact", "fast"])
@pytest.mark.parametrize("C,T,rows", [(1024, 8, [3000, 2500, 4001]), (512, 16, [700, 5, 0, 900, 3]),
                                      (256, 4, [1, 2, 3, 4000])])
def test_multi_device_segments_with_peer_halo(cuda, C, T, rows, flags):
    import torch
    ppf = ppf_mod()
    S = sum(rows)
    x = torch.empty((S, C), dtype=torch.complex64, device="cuda")
    ppf.synth(C, S * C, seed=C + T, out=x)
    coeffs = ppf.generate_prototype(C, T)
    f = ppf.EXACT if flags == "exact" else ppf.FAST
    with ppf.Plan(C, T, coeffs, flags=f) as p:
        want = p.fir_fft(x)
    torch.cuda.synchronize()
    plans = [ppf.Plan(C, T, coeffs, flags=f) for _ in rows]
    segs, outs, o = [], [], 0
    for r in rows:
        seg = torch.zeros((r + T - 1, C), dtype=torch.complex64, device="cuda")
        seg[:r] = x[o:o + r]
        segs.append(seg)
        outs.append(torch.empty((max(r, 1), C), dtype=torch.complex64, device="cuda"))
        o += r
    torch.cuda.synchronize()
    got = ppf.multi_fir_fft_device(plans, segs, rows, outs)
    for p in plans:
        p.close()
    assert sum(got) == S - T + 1
    cat = torch.cat([outs[g][:got[g]] for g in range(len(rows))])
    assert torch.equal(cat.view(torch.int64), want.view(torch.int64))


def test_host_pipeline_pinned_and_pageable(cuda, port):
    """ppfg_fir_fft with host buffers: multi-chunk double-buffered pipeline,
    pinned (torch pin_memory) and pageable (numpy) inputs give the same bytes."""
    import torch
    ppf = ppf_mod()
    C, T = 1024, 8
    S = (64 << 20) // (C * 8) * 2 + 777  # > 2 chunks of 64 MiB
    c = ppf.generate_prototype(C, T)
    x = ppf.synth(C, S * C, seed=4).reshape(S, C)
    with ppf.Plan(C, T, c, flags=ppf.EXACT) as p:
        a = p.fir_fft(x)
        xp = torch.from_numpy(x).pin_memory()
        b = p.fir_fft(xp)
    assert np.array_equal(bits(a), bits(b.numpy()))
    head = port.fir_fft(x[:3000], C, T, c.values)
    assert np.array_equal(bits(a[:3000 - T + 1]), bits(head))
    tail = port.fir_fft(x[-3000:], C, T, c.values)
    assert np.array_equal(bits(a[-(3000 - T + 1):]), bits(tail))


# ------------------------------------------------- detection
def _rel(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


@pytest.mark.parametrize("C,S", [(1024, 5000), (64, 3), (12, 700), (1, 10), (4096, 300)])
def test_mean_power_vs_oracle(cuda, port, C, S):
    """ppfg_mean_power == cmd_inspect's running sum up to summation order."""
    import torch
    ppf = ppf_mod()
    bins = uniform(np.random.default_rng(C + S), S * C).reshape(S, C)
    want = port.mean_power(bins, C)
    with ppf.Plan(C) as p:
        got = p.mean_power(bins)
        again = p.mean_power(bins)
        dev = p.mean_power(torch.from_numpy(bins).cuda())
        torch.cuda.synchronize()
    assert _rel(got, want) <= 1e-13
    assert np.array_equal(got, again)                 # deterministic
    assert np.array_equal(dev.cpu().numpy(), got)     # host and device paths agree


def test_mean_power_empty(cuda):
    ppf = ppf_mod()
    with ppf.Plan(16) as p:
        assert np.array_equal(p.mean_power(np.zeros(0, np.complex64)), np.zeros(16))


@pytest.mark.parametrize("C,T,flags", [(1024, 8, "fast"), (512, 8, "exact"), (1024, 4, "fast"),
                                       (512, 16, "fast"), (1024, 16, "fast"), (100, 4, "exact"),
                                       (2048, 8, "exact"), (128, 8, "fast"), (256, 8, "exact"),
                                       (256, 8, "fast"), (64, 8, "fast"), (64, 8, "exact"),
                                       (128, 8, "exact"), (1024, 4, "exact"), (4096, 8, "fast"),
                                       (1024, 8, "exact")])
def test_fir_fft_mean_power(cuda, port, C, T, flags):
    """Fused detection (bins never written where a detection kernel exists)
    == mean_power(fir_fft(x)) == the oracle's inspect of the oracle's bins."""
    ppf = ppf_mod()
    S = T - 1 + 148 * 8 * 2 + 37
    x = ppf.synth(C, S * C, seed=C + T)
    coeffs = port.generate_prototype(C, T, 9.0)
    f = ppf.FAST if flags == "fast" else ppf.EXACT
    with ppf.Plan(C, T, coeffs, flags=f) as p:
        fused = p.fir_fft_mean_power(x)
        bins = p.fir_fft(x)
        via_bins = p.mean_power(bins)
    want = port.mean_power(port.fir_fft(x, C, T, coeffs), C)
    # EXACT: FP64 accumulation, only the summation order differs; FAST: FP32
    # partial sums of 16 batches flushed into FP64 partials (fused.cuh)
    assert _rel(fused, via_bins) <= (1e-13 if flags == "exact" else 5e-6)
    if flags == "exact":
        assert _rel(fused, want) <= 1e-13              # bins bit-exact: only the sum order differs
    else:
        assert _rel(fused, want) <= 2e-5 * np.log2(C)  # FP32 FIR: |X|^2 inherits 2x its error


@pytest.mark.parametrize("C,T,flags", [(1024, 8, "fast"), (512, 8, "exact"), (2048, 8, "fast"),
                                       (1024, 16, "exact"), (1024, 4, "exact")])
def test_misaligned_device_views(cuda, port, C, T, flags):
    """Buffers that start 8 bytes past a 16-byte boundary (a view at an odd
    sample) cannot feed TMA: the plain-load kernels must take them, same results."""
    import torch
    ppf = ppf_mod()
    S = T - 1 + 300
    x = ppf.synth(C, S * C, seed=C + T)
    coeffs = port.generate_prototype(C, T, 9.0)
    want = port.fir_fft(x, C, T, coeffs).view(np.complex64)
    buf = torch.zeros(S * C + 1, dtype=torch.complex64, device=cuda)
    view = buf[1:]
    view.copy_(torch.from_numpy(x.reshape(-1)))
    assert view.data_ptr() % 16 == 8
    f = ppf.FAST if flags == "fast" else ppf.EXACT
    with ppf.Plan(C, T, coeffs, flags=f) as p:
        got = p.fir_fft(view).cpu().numpy()
        fir = p.fir(view).cpu().numpy()
        mp = p.fir_fft_mean_power(view)
        chan = p.channelize(view).cpu().numpy()
    torch.cuda.synchronize()
    if flags == "exact":
        assert np.array_equal(bits(got), bits(want))
    else:
        assert max_err_over_rms(got, want) <= 1e-5 * np.log2(C)
    assert np.array_equal(bits(fir), bits(port.fir(x, C, T, coeffs)))
    assert np.array_equal(bits(chan), bits(port.channelize(x, C)))
    assert _rel(mp.cpu().numpy(), port.mean_power(port.fir_fft(x, C, T, coeffs), C)) <= 2e-5 * np.log2(C)


# EXACT mode on the values where float <-> double conversion and the FFT's
# FP32 arithmetic are easiest to get wrong: zeros of both signs, float
# subnormals in and out, large magnitudes, and all-zero stretches (zero
# outputs) must come out bit-identical to the reference.
@pytest.mark.parametrize("C,T", [(1024, 8), (512, 8), (64, 8), (1024, 16), (256, 4), (2048, 8),
                                 (8, 8), (1024, 32)])
def test_exact_special_values_bitwise(cuda, port, C, T):
    ppf = ppf_mod()
    rng = np.random.default_rng(C + T)
    S = 300 + T
    x = uniform(rng, S * C).reshape(S, C).copy()
    xr = x.view(np.float32).reshape(S, C, 2)
    xr[5:5 + T + 3] = 0.0                                   # a zero stretch: zero outputs
    xr[40:60, :, 0] = -0.0                                  # negative zeros
    xr[70:90] *= np.float32(1e-39)                          # subnormal inputs
    xr[100:110] = rng.choice([1e-45, -1e-45, 3e-44], size=xr[100:110].shape).astype(np.float32)
    xr[120:130] *= np.float32(1e34)                         # large magnitudes (no FFT overflow)
    xr[140:150, :, 1] *= np.float32(1e-30)                  # results with tiny imaginary parts
    coeffs = port.generate_prototype(C, T, 9.0)
    want = port.fir_fft(x, C, T, coeffs).view(np.complex64).reshape(-1, C)
    for flags in (ppf.EXACT, ppf.EXACT | ppf.UNFUSED):
        with ppf.Plan(C, T, coeffs, flags=flags) as p:
            got = p.fir_fft(x)
        assert np.array_equal(bits(got), bits(want)), (C, T, flags, p.kernel_name)
