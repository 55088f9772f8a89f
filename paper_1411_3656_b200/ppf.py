"""Python mirror of the reference's public PPF API (proj/include/ppf/*.hpp) over
the C-ABI of libppfg.so — same function names, argument meaning and error
classes, so parity tests read like the reference's own tests.

Arrays: a block is a complex64 array of shape (n_spectra, n_channels) (or any
shape whose flat order is spectrum-major interleaved (re, im) f32 pairs).
numpy arrays (host) run the library's host-streamed path; torch tensors on a
CUDA device run in place on that device on torch's current stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

EXACT = 0
FAST = 1
UNFUSED = 2
CLUSTER = 4
K1_PREFETCH = 8  # comparison only: register-prefetch FIR kernel
FIR_LEGACY = 16  # comparison only: lane-window FIR kernels instead of K1b
L2X = 32  # also admit the L2-exchange fused kernels (K7) not taken by default
MEM_HOST = 0
MEM_DEVICE = 1

kDefaultBlockSpectra = 4096          # pipeline.hpp:16
kDefaultReferenceRate = 6_500_000_000  # pipeline.hpp:17
kDefaultKaiserBeta = 9.0             # coeff.hpp:17
kDefaultCutoffScale = 1.5            # coeff.hpp:24


# ---- errors.hpp ---------------------------------------------------------------
class PpfError(RuntimeError):
    status = -1


class config_error(PpfError, ValueError):                 # errors.hpp:11-13
    status = 1


class insufficient_history_error(config_error):          # errors.hpp:16-18
    status = 2


class unsupported_size_error(config_error):              # errors.hpp:21-23
    status = 3


class degenerate_filter_error(PpfError):                 # errors.hpp:26-28
    status = 4


class decode_error(PpfError):                            # errors.hpp:32-38
    status = 5

    def __init__(self, msg, byte_offset=0):
        super().__init__(msg)
        self.byte_offset = byte_offset


class io_error(PpfError):                                # errors.hpp:41-43
    status = 6


class cuda_error(PpfError):
    status = 7


class no_device_error(PpfError):
    status = 8


class domain_error(PpfError, ValueError):
    status = 9


_BY_STATUS = {c.status: c for c in (config_error, insufficient_history_error,
                                    unsupported_size_error, degenerate_filter_error,
                                    decode_error, io_error, cuda_error, no_device_error,
                                    domain_error)}


def _check(rc):
    if rc == 0:
        return
    lib = _lib.load()
    msg = lib.ppfg_last_error().decode(errors="replace")
    cls = _BY_STATUS.get(rc, PpfError)
    if cls is decode_error:
        raise decode_error(msg, lib.ppfg_last_error_offset())
    raise cls(msg)


# ---- coeff.hpp ------------------------------------------------------------------
@dataclass
class FilterCoefficients:                                # coeff.hpp:50-58
    n_channels: int
    n_taps: int
    values: np.ndarray = field(repr=False)

    def at(self, tap, channel):
        return float(self.values[tap * self.n_channels + channel])


def generate_prototype(n_channels, n_taps, beta=kDefaultKaiserBeta,
                       cutoff_scale=kDefaultCutoffScale) -> FilterCoefficients:
    """coeff.hpp:110-144 (Kaiser-windowed sinc, unit sum)."""
    lib = _lib.load()
    out = np.empty(n_channels * n_taps, np.float64)
    _check(lib.ppfg_generate_prototype(n_channels, n_taps, beta, cutoff_scale,
                                       out.ctypes.data_as(_lib.dp)))
    return FilterCoefficients(n_channels, n_taps, out)


def flops_for_fir(n_channels, n_taps, n_spectra_out):    # fir.hpp:49-52
    return _lib.load().ppfg_flops_for_fir(n_channels, n_taps, n_spectra_out)


def flops_for_dft(n_channels, n_spectra):                # dft.hpp:28-35
    return _lib.load().ppfg_flops_for_dft(n_channels, n_spectra)


# ---- buffers ----------------------------------------------------------------------
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _as_host(x):
    a = np.ascontiguousarray(x)
    if a.dtype == np.float32:
        a = a.view(np.complex64)
    if a.dtype != np.complex64:
        a = a.astype(np.complex64)
    return a


class _Buf:
    """(pointer, n_complex, mem kind, cuda stream) for numpy or torch input."""

    def __init__(self, x):
        self.keep = x
        if _is_torch(x):
            import torch
            if not x.is_contiguous():
                raise config_error("ppf: tensor must be contiguous")
            if x.dtype == torch.float32:
                n = x.numel() // 2
            elif x.dtype == torch.complex64:
                n = x.numel()
            else:
                raise config_error("ppf: tensor must be complex64 or interleaved float32")
            self.ptr = x.data_ptr()
            self.n = n
            if x.is_cuda:
                self.mem = MEM_DEVICE
                # torch's default stream is the legacy stream (handle 0); the C-ABI
                # reads NULL as "the plan's own stream", so name it explicitly
                # (cudaStreamLegacy == 0x1).
                self.stream = torch.cuda.current_stream(x.device).cuda_stream or 1
                self.device = x.device.index
            else:
                self.mem = MEM_HOST
                self.stream = None
                self.device = None
        else:
            a = _as_host(x)
            self.keep = a
            self.ptr = a.ctypes.data
            self.n = a.size
            self.mem = MEM_HOST
            self.stream = None
            self.device = None


def _empty_like(x, n_complex, shape):
    if _is_torch(x):
        import torch
        return torch.empty(shape, dtype=torch.complex64, device=x.device)
    return np.empty(shape, np.complex64)


# ---- plans --------------------------------------------------------------------------
class Plan:
    """Device state for one (C, T) channelizer (ppfg_plan_create)."""

    def __init__(self, n_channels, n_taps=0, coeffs=None, flags=EXACT, device=0):
        lib = _lib.load()
        self.n_channels = int(n_channels)
        self.n_taps = int(n_taps)
        self.flags = flags
        self.device = device
        vals = None
        if n_taps:
            if coeffs is None:
                raise config_error("fir: malformed coefficient set")
            v = coeffs.values if isinstance(coeffs, FilterCoefficients) else coeffs
            vals = np.ascontiguousarray(v, np.float64)
            if vals.size != self.n_channels * self.n_taps:
                raise config_error("fir: malformed coefficient set")
            if isinstance(coeffs, FilterCoefficients) and (
                    coeffs.n_channels != n_channels or coeffs.n_taps != n_taps):
                raise config_error("fir: input channel count does not match coefficients")
        self._vals = vals
        h = C.c_void_p()
        _check(lib.ppfg_plan_create(C.byref(h), self.n_channels, self.n_taps,
                                    vals.ctypes.data_as(_lib.dp) if vals is not None else None,
                                    flags, device))
        self._h = h
        self._lib = lib

    @property
    def handle(self):
        return self._h

    @property
    def kind(self):
        return self._lib.ppfg_fir_fft_kind(self._h)

    @property
    def kernel_name(self):
        """The fir_fft kernel, as ncu names it (ppfg_fir_fft_kernel_name)."""
        return self._lib.ppfg_fir_fft_kernel_name(self._h).decode()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ppfg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _rows(self, b):
        if b.n % self.n_channels != 0 or b.n == 0:
            raise config_error("SampleBlock: sample count must be a positive multiple of "
                               "n_channels")
        return b.n // self.n_channels

    def _call(self, fn, x, out, n_out_rows, *extra, rows=None):
        b = _Buf(x)
        s_in = self._rows(b) if rows is None else rows
        if out is None:
            out = _empty_like(x, n_out_rows(s_in) * self.n_channels,
                              (max(n_out_rows(s_in), 0), self.n_channels))
        o = _Buf(out)
        if o.mem != b.mem:
            raise config_error("ppf: input and output must live in the same memory")
        if max(n_out_rows(s_in), 0) * self.n_channels > o.n:
            raise config_error("ppf: output buffer too small")
        _check(fn(self._h, b.ptr, s_in, o.ptr, *extra, b.mem, b.stream))
        return out

    def fir(self, x, out=None):
        """ppf_fir_optimized (fir.hpp:158-212), bit-exact."""
        return self._call(self._lib.ppfg_fir, x, out, lambda s: s - self.n_taps + 1)

    def fir_reference(self, x, out=None):
        """ppf_fir_reference (fir.hpp:123-151), bit-exact."""
        return self._call(self._lib.ppfg_fir_reference_order, x, out,
                          lambda s: s - self.n_taps + 1)

    def channelize(self, x, out=None, fft_fallback=True):
        """channelize_block (dft.hpp:175-235)."""
        b = _Buf(x)
        if b.n % self.n_channels != 0:
            raise config_error("channelize_block: malformed filtered block")
        rows = b.n // self.n_channels
        if out is None:
            out = _empty_like(x, rows * self.n_channels, (rows, self.n_channels))
        if rows == 0:
            return out
        o = _Buf(out)
        _check(self._lib.ppfg_channelize(self._h, b.ptr, rows, o.ptr, int(bool(fft_fallback)),
                                         b.mem, b.stream))
        return out

    def fir_fft(self, x, out=None):
        """channelize_block(ppf_fir_optimized(x)) — fused where available."""
        return self._call(self._lib.ppfg_fir_fft, x, out, lambda s: s - self.n_taps + 1)

    def _power(self, fn, x, rows):
        b = _Buf(x)
        if _is_torch(x):
            import torch
            out = torch.empty(self.n_channels, dtype=torch.float64, device=x.device)
            optr = out.data_ptr()
        else:
            out = np.empty(self.n_channels, np.float64)
            optr = out.ctypes.data
        _check(fn(self._h, b.ptr, rows(b), optr, b.mem, b.stream))
        return out

    def mean_power(self, bins):
        """Per-channel mean power of channelized spectra, as `ppf inspect`
        computes it (cmd_inspect, cli.hpp:307-317): float64[C]."""
        def rows(b):
            if b.n % self.n_channels:
                raise config_error("inspect: malformed channelized block")
            return b.n // self.n_channels
        return self._power(self._lib.ppfg_mean_power, bins, rows)

    def fir_fft_mean_power(self, x):
        """mean_power(fir_fft(x)) without writing the bins (fused detection)."""
        return self._power(self._lib.ppfg_fir_fft_mean_power, x, self._rows)


# ---- one-shot reference-style API ---------------------------------------------------
def _coeff_plan(coeffs: FilterCoefficients, flags=EXACT, device=0):
    return Plan(coeffs.n_channels, coeffs.n_taps, coeffs, flags, device)


def _check_block(x, n_channels):
    a = x if _is_torch(x) else _as_host(x)
    n = a.numel() if _is_torch(a) else a.size
    if n_channels == 0:
        raise config_error("SampleBlock: n_channels must be >= 1")
    if n == 0 or n % n_channels:
        raise config_error("SampleBlock: sample count must be a positive multiple of n_channels")
    return a


def ppf_fir_optimized(block, coeffs: FilterCoefficients, workers=1, n_channels=None):
    """fir.hpp:158-212. `workers` is kept for signature compatibility; the
    decomposition is over CUDA threads and never changes the result."""
    if workers == 0:
        raise config_error("fir: workers must be >= 1")
    nc = coeffs.n_channels if n_channels is None else n_channels
    a = _check_block(block, nc)
    if nc != coeffs.n_channels:
        raise config_error("fir: input channel count does not match coefficients")
    with _coeff_plan(coeffs) as p:
        return p.fir(a)


def ppf_fir_reference(block, coeffs: FilterCoefficients, n_channels=None):
    """fir.hpp:123-151."""
    nc = coeffs.n_channels if n_channels is None else n_channels
    a = _check_block(block, nc)
    if nc != coeffs.n_channels:
        raise config_error("fir: input channel count does not match coefficients")
    with _coeff_plan(coeffs) as p:
        return p.fir_reference(a)


def channelize_block(filtered, n_channels, fft_fallback=True, workers=1):
    """dft.hpp:175-235."""
    if n_channels == 0:
        raise config_error("channelize_block: n_channels must be >= 1")
    if workers == 0:
        raise config_error("channelize_block: workers must be >= 1")
    with Plan(n_channels, 0) as p:
        return p.channelize(filtered, fft_fallback=fft_fallback)


def fft(x):
    """dft.hpp:160-169 (one row, power-of-two length)."""
    a = _as_host(x).reshape(-1)
    out = np.empty_like(a)
    _check(_lib.load().ppfg_fft(a.ctypes.data, a.size, out.ctypes.data))
    return out


def dft_naive(x):
    """dft.hpp:39-66 (one row, any length)."""
    a = _as_host(x).reshape(-1)
    out = np.empty_like(a)
    _check(_lib.load().ppfg_dft_naive(a.ctypes.data, a.size, out.ctypes.data))
    return out


# ---- streaming (pipeline.hpp) ---------------------------------------------------------
@dataclass
class StreamStateView:                                   # pipeline.hpp:43-49
    spectra_processed: int = 0
    bytes_in: int = 0
    bytes_out: int = 0
    dropped_samples: int = 0


class Stream:
    """Device-resident process_stream state: push raw bytes, get spectra bytes."""

    def __init__(self, plan: Plan, block_spectra=kDefaultBlockSpectra, zero_prime=False,
                 fft_fallback=True):
        self.plan = plan
        self.block_spectra = block_spectra
        self._lib = _lib.load()
        h = C.c_void_p()
        _check(self._lib.ppfg_stream_open(C.byref(h), plan.handle, block_spectra,
                                          int(zero_prime), int(fft_fallback)))
        self._h = h

    def push(self, data: bytes) -> bytes:
        row = self.plan.n_channels * 8
        cap = (len(data) // row + 2 + self.block_spectra + self.plan.n_taps) * row
        out = np.empty(cap, np.uint8)
        n = C.c_uint64(0)
        src = np.frombuffer(data, np.uint8) if len(data) else np.zeros(1, np.uint8)
        _check(self._lib.ppfg_stream_push(self._h, src.ctypes.data, len(data), out.ctypes.data,
                                          cap, C.byref(n)))
        return out[: n.value].tobytes()

    def close(self) -> StreamStateView:
        st = _lib.StreamState()
        _check(self._lib.ppfg_stream_close(self._h, C.byref(st)))
        return StreamStateView(st.spectra_processed, st.bytes_in, st.bytes_out,
                               st.dropped_samples)

    def destroy(self):
        if getattr(self, "_h", None):
            self._lib.ppfg_stream_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def process_stream(n_channels, n_taps, source, sink, block_spectra=kDefaultBlockSpectra,
                   zero_prime=False, coefficients: FilterCoefficients | None = None,
                   fft_fallback=True, beta=kDefaultKaiserBeta, flags=EXACT, device=0):
    """pipeline.hpp:89-200: read raw LE f32 pairs from `source` (file-like,
    .read(n)), write channelized spectra to `sink` (.write(bytes))."""
    if n_channels == 0:
        raise config_error("config: n_channels must be >= 1")
    if n_taps == 0:
        raise config_error("config: n_taps must be >= 1")
    if block_spectra < n_taps:
        raise config_error("config: block_spectra must be >= n_taps")
    if coefficients is not None:
        if coefficients.n_channels != n_channels or coefficients.n_taps != n_taps:
            raise config_error("process_stream: supplied coefficients do not match the config")
        coeffs = coefficients
    else:
        coeffs = generate_prototype(n_channels, n_taps, beta)
    lib = _lib.load()
    err = {}

    def _read(ctx, buf, n):
        try:
            data = source.read(n)
        except Exception as e:  # source failure -> decode_error at the current offset
            err["read"] = e
            return -1
        C.memmove(buf, data, len(data))
        return len(data)

    def _write(ctx, buf, n):
        try:
            sink.write(C.string_at(buf, n))
            return 0
        except Exception as e:
            err["write"] = e
            return 1

    rfn, wfn = _lib.READ_FN(_read), _lib.WRITE_FN(_write)
    st = _lib.StreamState()
    with Plan(n_channels, n_taps, coeffs, flags, device) as p:
        rc = lib.ppfg_process_stream(p.handle, block_spectra, int(zero_prime),
                                     int(fft_fallback), rfn, None, wfn, None, C.byref(st))
    _check(rc)
    return StreamStateView(st.spectra_processed, st.bytes_in, st.bytes_out, st.dropped_samples)


# ---- sharding + synthetic input ---------------------------------------------------------
def shard_range(n_spectra_in, n_taps, rank, world):
    """(in_begin, in_count, out_begin, out_count) of shard `rank`."""
    v = [C.c_uint64() for _ in range(4)]
    _check(_lib.load().ppfg_shard_range(n_spectra_in, n_taps, rank, world,
                                        *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def multi_fir_fft(host_in, coeffs: FilterCoefficients, devices, flags=EXACT):
    """ppfg_multi_fir_fft: shards over `devices`, one host thread each."""
    a = _as_host(host_in).reshape(-1)
    C_, T = coeffs.n_channels, coeffs.n_taps
    s_in = a.size // C_
    out = np.empty((s_in - T + 1, C_), np.complex64)
    devs = (C.c_int * len(devices))(*devices)
    vals = np.ascontiguousarray(coeffs.values, np.float64)
    _check(_lib.load().ppfg_multi_fir_fft(C_, T, vals.ctypes.data_as(_lib.dp), flags, devs,
                                          len(devices), a.ctypes.data, s_in, out.ctypes.data))
    return out


def multi_fir_fft_device(plans, segments, seg_rows, outs):
    """ppfg_multi_fir_fft_device (halo from the peer): segment g is
    a CUDA tensor on plans[g]'s device holding seg_rows[g] input spectra plus
    n_taps - 1 spare rows; returns the output spectra count per segment (outs[g]
    receives them)."""
    n = len(plans)
    if not (len(segments) == len(seg_rows) == len(outs) == n):
        raise config_error("multi_fir_fft_device: one segment, row count and output per plan")
    ph = (_lib.vp * n)(*[p._h.value for p in plans])
    ins = (_lib.vp * n)(*[_Buf(x).ptr for x in segments])
    os_ = (_lib.vp * n)(*[_Buf(y).ptr for y in outs])
    rows = (_lib.u64 * n)(*seg_rows)
    got = (_lib.u64 * n)()
    _check(_lib.load().ppfg_multi_fir_fft_device(ph, n, ins, rows, os_, got))
    return [int(v) for v in got]


def synth(n_channels, n_samples, seed=1, first_sample=0, out=None, device=0, stream=None):
    """Counter-based tone + noise (ppfg_synth). numpy out -> host generator,
    torch CUDA out -> device kernel; identical bytes."""
    lib = _lib.load()
    if out is None:
        out = np.empty(n_samples, np.complex64)
    b = _Buf(out)
    if b.n < n_samples:
        raise config_error("synth: output too small")
    s = stream if stream is not None else b.stream
    _check(lib.ppfg_synth(n_channels, seed, first_sample, n_samples, b.ptr, b.mem,
                          b.device if b.device is not None else device, s))
    return out


def kernel_launches():
    return _lib.load().ppfg_kernel_launches()
