"""Out-of-bounds write guards for every kernel family (compute-sanitizer is
closed on this GPU pool): the output of each call is a view
in the middle of a larger device buffer whose head and tail are filled with a
canary pattern; after the call the canaries must be intact and the output
must equal the reference's. The input is likewise a view whose neighbouring
rows hold NaNs: a kernel that reads a row outside its input would poison the
result, which the parity check catches. Ragged sizes (tails that do not fill
a batch, a chunk or a warp) are included on purpose."""
import numpy as np
import pytest

from conftest import bits, max_err_over_rms

pytestmark = pytest.mark.gpu

GUARD = 4096          # canary rows on each side (complex64 rows of C)
CANARY = 0x7FC0DEAD   # a NaN payload no kernel produces


def _ppf():
    from paper_1411_3656_b200 import ppf
    return ppf


CASES = [
    # (C, T, flags, S_in, what)
    (1024, 8, "fast", 1000, "K3 SKA shape, HS + TRIV"),
    (512, 8, "exact", 777, "K3 FP64"),
    (256, 4, "fast", 513, "K3, several FIR groups"),
    (1024, 16, "fast", 600, "K3s 2-CTA cluster"),
    (1024, 8, "exact", 420, "K3s FP64"),
    (4096, 8, "fast", 150, "K3s 4-CTA cluster"),
    (8, 8, "exact", 3001, "K6 tiny C"),
    (32, 32, "fast", 2000, "K6 T = 32"),
    (1024, 32, "fast", 900, "unfused K1b + K3(T=1)"),
    (1024, 64, "exact", 500, "unfused K1b FP64"),
    (8192, 8, "fast", 40, "K1t + K2n"),
    (100, 4, "exact", 90, "K1 + K4 dft_naive"),
    (1024, 32, "fast+l2x", 1300, "K7 L2 exchange"),
    (8192, 8, "exact+l2x", 300, "K7 at C = 8192"),
]


@pytest.mark.parametrize("C,T,mode,S,what", CASES, ids=[c[4] for c in CASES])
def test_no_write_outside_the_output(cuda, port, C, T, mode, S, what):
    import torch
    ppf = _ppf()
    flags = (ppf.FAST if mode.startswith("fast") else ppf.EXACT) | (ppf.L2X if "l2x" in mode else 0)
    coeffs = port.generate_prototype(C, T, 9.0)
    x_host = ppf.synth(C, S * C, seed=C + T + S).reshape(S, C)
    want = port.fir_fft(x_host, C, T, coeffs).view(np.complex64).reshape(-1, C)
    S_out = S - T + 1
    # input view with NaN rows around it
    xin = torch.full((S + 2 * GUARD, C), float("nan"), dtype=torch.complex64, device=cuda)
    xin[GUARD:GUARD + S] = torch.from_numpy(x_host).to(cuda)
    # output view inside canaries
    buf = torch.empty((S_out + 2 * GUARD, C), dtype=torch.complex64, device=cuda)
    torch.view_as_real(buf).view(torch.int32).fill_(CANARY)
    y = buf[GUARD:GUARD + S_out]
    with ppf.Plan(C, T, coeffs, flags=flags) as p:
        p.fir_fft(xin[GUARD:GUARD + S], out=y)
        torch.cuda.synchronize()
    raw = torch.view_as_real(buf).view(torch.int32)
    assert bool((raw[:GUARD] == CANARY).all()), f"{what}: write before the output"
    assert bool((raw[GUARD + S_out:] == CANARY).all()), f"{what}: write after the output"
    got = y.cpu().numpy()
    if mode.startswith("exact"):
        assert np.array_equal(bits(got), bits(want)), what
    else:
        assert max_err_over_rms(got, want) <= 1e-5 * np.log2(C), what


@pytest.mark.parametrize("C,T,mode,S", [(1024, 8, "fast", 1000), (512, 8, "exact", 700),
                                        (2048, 8, "fast", 300), (256, 16, "fast", 450)])
def test_detection_partials_stay_inside(cuda, port, C, T, mode, S):
    """Fused detection writes per-CTA partials into a plan-owned buffer; the
    caller's C doubles are the only caller memory written."""
    import torch
    ppf = _ppf()
    flags = ppf.FAST if mode == "fast" else ppf.EXACT
    coeffs = port.generate_prototype(C, T, 9.0)
    x = torch.from_numpy(ppf.synth(C, S * C, seed=S).reshape(S, C)).to(cuda)
    with ppf.Plan(C, T, coeffs, flags=flags) as p:
        a = p.fir_fft_mean_power(x)
        b = p.fir_fft_mean_power(x)
        torch.cuda.synchronize()
    assert a.shape == (C,) and torch.equal(a, b)   # deterministic, repeatable
    assert bool(torch.isfinite(a).all())


@pytest.mark.parametrize("C,S", [(64, 1000), (256, 333), (1024, 77), (2048, 5), (4096, 9), (8192, 3)])
def test_channelize_writes_only_its_rows(cuda, port, C, S):
    """channelize_block (K2n row tiles, ragged last tiles; shared or global
    last-pass twiddles): the output view sits between canary rows, the input
    view between NaN rows; in place as well."""
    import torch
    ppf = _ppf()
    x_host = ppf.synth(C, S * C, seed=C + S).reshape(S, C)
    want = port.channelize(x_host, C).view(np.complex64).reshape(S, C)
    xin = torch.full((S + 2 * GUARD, C), float("nan"), dtype=torch.complex64, device=cuda)
    xin[GUARD:GUARD + S] = torch.from_numpy(x_host).to(cuda)
    buf = torch.empty((S + 2 * GUARD, C), dtype=torch.complex64, device=cuda)
    torch.view_as_real(buf).view(torch.int32).fill_(CANARY)
    with ppf.Plan(C, 1, port.generate_prototype(C, 1, 9.0)) as p:
        p.channelize(xin[GUARD:GUARD + S], out=buf[GUARD:GUARD + S])
        p.channelize(xin[GUARD:GUARD + S], out=xin[GUARD:GUARD + S])   # in place
        torch.cuda.synchronize()
    raw = torch.view_as_real(buf).view(torch.int32)
    assert bool((raw[:GUARD] == CANARY).all()) and bool((raw[GUARD + S:] == CANARY).all())
    assert bool(torch.isnan(xin[:GUARD]).all()) and bool(torch.isnan(xin[GUARD + S:]).all())
    assert np.array_equal(bits(buf[GUARD:GUARD + S].cpu().numpy()), bits(want))
    assert np.array_equal(bits(xin[GUARD:GUARD + S].cpu().numpy()), bits(want))
