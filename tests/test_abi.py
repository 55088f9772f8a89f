"""CPU-side checks of the product library: it builds for sm_100a, loads,
exports every symbol include/ppfg.h declares, validates arguments without a
GPU, and its host-side logic (prototype design, sharding, synthetic input,
FLOP conventions) matches the reference. No kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ppfg.h")).read()
    return sorted(set(re.findall(r"\b(ppfg_[a-z0-9_]+)\s*\(", src)) - {"ppfg_read_fn",
                                                                     "ppfg_write_fn"})


def test_library_exports_every_header_symbol():
    from paper_1411_3656_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signatures out of sync with ppfg.h"


def test_library_is_sm100a_only():
    import subprocess
    from paper_1411_3656_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.so_path()], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_device_is_a_loud_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1411_3656_b200 import ppf
    with pytest.raises(ppf.no_device_error):
        ppf.Plan(8, 4, np.ones(32))


def test_prototype_matches_reference_bitwise(golden):
    from paper_1411_3656_b200 import ppf
    for i, (C, T, b) in enumerate(golden["protos"]):
        got = ppf.generate_prototype(int(C), int(T), float(b)).values
        assert np.array_equal(got.view(np.uint64), golden[f"proto{i}"].view(np.uint64))
    with pytest.raises(ppf.config_error):
        ppf.generate_prototype(0, 4)
    with pytest.raises(ppf.config_error):
        ppf.generate_prototype(4, 4, beta=-1.0)


def test_flop_conventions():
    from paper_1411_3656_b200 import ppf
    assert ppf.flops_for_fir(256, 8, 1000) == 8_192_000
    assert ppf.flops_for_dft(1024, 1) == 51_200
    assert ppf.flops_for_dft(6, 10) == 2_880


@pytest.mark.parametrize("S_in,T,world", [(100, 8, 1), (100, 8, 2), (793457, 8, 8), (17, 16, 4),
                                          (10, 3, 8), (64, 1, 3)])
def test_shard_ranges_tile_the_output(S_in, T, world):
    from paper_1411_3656_b200 import ppf
    S_out = S_in - T + 1
    cover = []
    for r in range(world):
        ib, ic, ob, oc = ppf.shard_range(S_in, T, r, world)
        assert ib == ob
        assert ic == (oc + T - 1 if oc else 0)
        assert ib + ic <= S_in
        cover.extend(range(ob, ob + oc))
    assert cover == list(range(S_out))
    with pytest.raises(ppf.insufficient_history_error):
        ppf.shard_range(T - 1, T, 0, 1) if T > 1 else ppf.shard_range(0, 1, 0, 1)


def test_synth_host_is_deterministic_and_tone_plus_noise():
    from paper_1411_3656_b200 import ppf
    C = 64
    a = ppf.synth(C, 4096, seed=3)
    b = ppf.synth(C, 2048, seed=3, first_sample=2048)
    assert np.array_equal(a[2048:].view(np.uint32), b.view(np.uint32))
    noise = a - np.exp(2j * np.pi * (C / 8 + 0.3) * np.arange(4096) / C).astype(np.complex64)
    assert abs(noise.real.std() - 1.0) < 0.05 and abs(noise.imag.std() - 1.0) < 0.05
    assert abs(noise.mean()) < 0.05


def test_oracle_synth_equals_the_library_generator():
    """The reference arm of bench.py feeds the reference from the oracle's copy
    of the synthetic generator (it must not load libppfg.so); its bytes must be
    the product's (which the GPU tests pin to the device generator)."""
    import oracle
    from paper_1411_3656_b200 import ppf
    for C, n, first, seed in [(1024, 1 << 18, 0, 1), (512, 12345, 777, 3), (8192, 5000, 10**12, 9)]:
        a = oracle.port().synth(C, n, seed=seed, first_sample=first)
        b = ppf.synth(C, n, seed=seed, first_sample=first)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (C, n, first)


def test_kernel_name_is_exported():
    from paper_1411_3656_b200 import _lib
    lib = _lib.load()
    assert lib.ppfg_fir_fft_kernel_name(None) == b""


def test_new_entry_points_validate_arguments_without_a_gpu():
    """ppfg_multi_fir_fft_device and ppfg_process_stream reject null arguments
    before touching a device (status codes of include/ppfg.h)."""
    import ctypes as C
    from paper_1411_3656_b200 import _lib
    lib = _lib.load()
    CONFIG_ERROR = 1   # PPFG_CONFIG_ERROR
    rows = (C.c_uint64 * 1)(8)
    got = (C.c_uint64 * 1)()
    assert lib.ppfg_multi_fir_fft_device(None, 1, None, rows, None, got) == CONFIG_ERROR
    assert lib.ppfg_multi_fir_fft_device(None, 0, None, None, None, None) == CONFIG_ERROR
    assert b"null" in lib.ppfg_last_error()
    st = _lib.StreamState()
    assert lib.ppfg_process_stream(None, 4096, 0, 1, _lib.READ_FN(0), None, _lib.WRITE_FN(0), None,
                                   C.byref(st)) == CONFIG_ERROR


@pytest.mark.parametrize("n,off", [(0, 0), (1, 1), (300_001, 3), ((1 << 20) + 3, 1),
                                   ((5 << 20) + 17, 5), ((33 << 20) + 5, 7)])
def test_host_copy_pool_copies_every_byte(n, off):
    """ppfg_host_copy (the pageable staging copy: a thread pool, streaming
    stores for large pieces, hostcopy.cpp) on unaligned ragged sizes — no GPU
    involved. The bytes around the destination stay untouched."""
    from paper_1411_3656_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(n)
    src = rng.integers(0, 256, n + 64, dtype=np.uint8)
    dst = np.full(n + 64, 0xA5, np.uint8)
    rc = lib.ppfg_host_copy(dst.ctypes.data + off, src.ctypes.data + (off * 3) % 32, n)
    assert rc == 0
    assert np.array_equal(dst[off:off + n], src[(off * 3) % 32:(off * 3) % 32 + n])
    assert (dst[:off] == 0xA5).all() and (dst[off + n:] == 0xA5).all()
