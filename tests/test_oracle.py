"""Pin the CPU restatement (oracle/ppf_oracle.c) before trusting it:
  * bit-for-bit against the golden vectors produced by the UNMODIFIED reference
    (tests/golden/make_golden.py),
  * bit-for-bit against the compiled reference itself on fresh random cases
    (where oracle/_ref exists),
  * against the known-answer values the reference's own tests hard-code."""
import numpy as np
import pytest

from conftest import bits, uniform


def test_port_fir_matches_golden(port, golden):
    for i in range(int(golden["n_fir"])):
        C, T = int(golden[f"fir{i}_C"]), int(golden[f"fir{i}_T"])
        x, c = golden[f"fir{i}_x"], golden[f"fir{i}_coeffs"]
        assert np.array_equal(bits(port.fir(x, C, T, c)), bits(golden[f"fir{i}_y"])), (C, T)
        assert np.array_equal(bits(port.fir(x, C, T, c, reference_order=True)),
                              bits(golden[f"fir{i}_y_ref"])), (C, T)


def test_port_fft_matches_golden(port, golden):
    for n in golden["fft_sizes"]:
        n = int(n)
        assert np.array_equal(bits(port.channelize(golden[f"fft{n}_x"], n)),
                              bits(golden[f"fft{n}_y"])), n
    for n in golden["dft_sizes"]:
        n = int(n)
        assert np.array_equal(bits(port.channelize(golden[f"dft{n}_x"], n)),
                              bits(golden[f"dft{n}_y"])), n


def test_port_fused_and_prototype_match_golden(port, golden):
    for i in range(int(golden["n_ff"])):
        C, T = int(golden[f"ff{i}_C"]), int(golden[f"ff{i}_T"])
        got = port.fir_fft(golden[f"ff{i}_x"], C, T, golden[f"ff{i}_coeffs"])
        assert np.array_equal(bits(got), bits(golden[f"ff{i}_y"])), (C, T)
    for i, (C, T, b) in enumerate(golden["protos"]):
        got = port.generate_prototype(int(C), int(T), float(b))
        assert np.array_equal(got.view(np.uint64), golden[f"proto{i}"].view(np.uint64))


def test_port_stream_matches_golden(port, golden):
    src = golden["stream_x"].tobytes()
    c = port.generate_prototype(8, 8, 9.0)
    for bs in (8, 100, 999, 4096):
        y, st = port.process_stream(src, 8, 8, bs, c)
        assert y == golden["stream_y"].tobytes(), bs
        assert [st.spectra_processed, st.bytes_in, st.bytes_out, st.dropped_samples] == \
            list(golden["stream_state"])
    y, st = port.process_stream(src, 8, 8, 64, c, zero_prime=True)
    assert y == golden["stream_zp_y"].tobytes()


def test_port_matches_compiled_reference_random(port, ref):
    rng = np.random.default_rng(7)
    for trial in range(60):
        C = int(rng.choice([1, 2, 3, 8, 64, 100, 256, 1024]))
        T = int(rng.choice([1, 2, 3, 8, 16, 32]))
        S = T + int(rng.integers(0, 21))
        x = uniform(rng, S * C)
        c = ref.generate_prototype(C, T, float(rng.uniform(0, 12)))
        assert np.array_equal(bits(port.fir(x, C, T, c)), bits(ref.fir(x, C, T, c, workers=4)))
        assert np.array_equal(bits(port.fir_fft(x, C, T, c)),
                              bits(ref.fir_fft(x, C, T, c, workers=2)))


def test_port_decode_error_offset(port, ref, golden):
    src = golden["stream_x"].tobytes()
    c = port.generate_prototype(8, 8, 9.0)
    bad = src[: 8 * 8 * 10] + b"\x01\x02\x03"
    for impl in (port, ref):
        with pytest.raises(Exception) as e:
            impl.process_stream(bad, 8, 8, 16, c)
        assert e.value.status == 5 and e.value.offset == 8 * 8 * 10


def test_known_answers(port):
    # coeff_test.cpp:180-189 frozen values
    v = port.generate_prototype(4, 8, 9.0)
    for k, want in [(0, -1.043256612690511e-05), (5, -0.0006421604682661697),
                    (13, 0.022228516434272306), (15, 0.3521187570439705),
                    (16, 0.3521187570439705), (31, -1.043256612690511e-05)]:
        assert abs(v[k] - want) / abs(want) < 1e-9
    assert list(port.generate_prototype(2, 1, 0.0)) == [0.5, 0.5]  # coeff_test.cpp:171-176
    # fir_test.cpp:259-263, dft_test.cpp:199-206
    assert port.flops_for_fir(1, 1, 1) == 4
    assert port.flops_for_fir(256, 8, 1000) == 8_192_000
    assert port.flops_for_fir(1024, 16, 1) == 65_536
    assert [port.flops_for_dft(*a) for a in [(1, 5), (1024, 1), (8, 100), (3, 2), (6, 10)]] == \
        [0, 51_200, 12_000, 144, 2_880]
    # dft_test.cpp:32-40: constant row -> bin 0
    y = port.dft_naive(np.ones(4, np.complex64))
    assert abs(y[0] - 4.0) < 1e-6 and np.all(np.abs(y[2:]) < 1e-6)
    # fir_test.cpp:73-82: T=1 unit coefficients is the identity
    rng = np.random.default_rng(101)
    x = uniform(rng, 60)
    assert np.array_equal(bits(port.fir(x, 6, 1, np.ones(6))), bits(x))
    # bessel_i0 known values (SPEC.md: I0(1) ~ 1.2660658778, I0(2) ~ 2.2795853023)
    assert abs(port.bessel_i0(1.0) - 1.2660658778) < 1e-9
    assert abs(port.bessel_i0(2.0) - 2.2795853023) < 1e-9


def test_port_impulse_orientation(port):
    # fir_test.cpp:87-110: an impulse at spectrum p reproduces h[p - s][c]
    rng = np.random.default_rng(103)
    C, T, S, ch, pos = 4, 5, 12, 2, 6
    c = rng.uniform(0.25, 1.75, C * T)
    x = np.zeros(S * C, np.complex64)
    x[pos * C + ch] = 1.0
    y = port.fir(x, C, T, c).view(np.complex64).reshape(S - T + 1, C)
    for s in range(S - T + 1):
        for cc in range(C):
            if cc == ch and s + T > pos >= s:
                assert y[s, cc] == np.float32(c[(pos - s) * C + cc])
            else:
                assert y[s, cc] == 0


def test_port_mean_power_is_the_inspect_running_sum(port):
    """cmd_inspect (cli.hpp:307-317): one running double sum per channel, in
    spectrum order, of (double)re^2 + (double)im^2, then / n."""
    rng = np.random.default_rng(5)
    C, S = 6, 37
    x = uniform(rng, S * C).reshape(S, C)
    want = np.zeros(C)
    for s in range(S):
        for c in range(C):
            re, im = float(x[s, c].real), float(x[s, c].imag)
            want[c] += re * re + im * im
    want /= S
    got = port.mean_power(x, C)
    assert np.array_equal(got, want)
    assert np.array_equal(port.mean_power(np.zeros(0, np.complex64), C), np.zeros(C))
