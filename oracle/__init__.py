"""CPU checkers for the PPF hot path — TEST INFRASTRUCTURE ONLY.

`port()` loads the C restatement (oracle/ppf_oracle.c, builds anywhere with
gcc). `reference()` loads the unmodified reference compiled from
/root/reference (oracle/_ref, built here by oracle/Makefile; the .so files
travel to the GPU box). Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs may import this package. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_PORT_SO = os.path.join(HERE, "_build", "libppforacle.so")
_REF_DIR = os.path.join(HERE, "_ref")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_sz = C.c_size_t

STATUS_NAMES = {0: "ok", 1: "config_error", 2: "insufficient_history_error",
                3: "unsupported_size_error", 4: "degenerate_filter_error",
                5: "decode_error", 6: "io_error", 9: "domain_error", 99: "other"}


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class StreamState(C.Structure):
    _fields_ = [("spectra_processed", C.c_uint64), ("bytes_in", C.c_uint64),
                ("bytes_out", C.c_uint64), ("dropped_samples", C.c_uint64),
                ("error_offset", C.c_uint64)]


def build_port():
    subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])


def build_ref():
    """Compile oracle/_ref from /root/reference (only where it exists)."""
    if not os.path.isdir("/root/reference/proj/include"):
        return False
    subprocess.check_call(["make", "-s", "-C", HERE, "ref"],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    return True


def _cf(a):
    a = np.ascontiguousarray(a)
    if np.iscomplexobj(a):
        return np.ascontiguousarray(a, dtype=np.complex64).view(np.float32)
    return np.ascontiguousarray(a, dtype=np.float32)


class _Port:
    def __init__(self):
        if not os.path.exists(_PORT_SO):
            build_port()
        L = self.lib = C.CDLL(_PORT_SO)
        L.ppfo_generate_prototype.argtypes = [_sz, _sz, C.c_double, C.c_double, _f64p]
        L.ppfo_fir.argtypes = [_f32p, _sz, _sz, _sz, _f64p, _f32p, C.c_int]
        L.ppfo_dft_naive.argtypes = [_f32p, _sz, _f32p]
        L.ppfo_fft.argtypes = [_f32p, _sz]
        L.ppfo_channelize.argtypes = [_f32p, _sz, _sz, C.c_int, _f32p]
        L.ppfo_fir_fft.argtypes = [_f32p, _sz, _sz, _sz, _f64p, C.c_int, _f32p]
        L.ppfo_mean_power.argtypes = [_f32p, _sz, _sz, _f64p]
        L.ppfo_process_stream.argtypes = [_sz, _sz, _sz, C.c_int, C.c_int, C.c_void_p, _u8p, _sz,
                                          _u8p, C.POINTER(StreamState)]
        L.ppfo_bessel_i0.argtypes = [C.c_double, C.POINTER(C.c_int)]
        L.ppfo_bessel_i0.restype = C.c_double
        L.ppfo_flops_for_fir.argtypes = [_sz, _sz, _sz]
        L.ppfo_flops_for_fir.restype = C.c_uint64
        L.ppfo_flops_for_dft.argtypes = [_sz, _sz]
        L.ppfo_flops_for_dft.restype = C.c_uint64
        L.ppfo_synth.argtypes = [_sz, C.c_uint64, C.c_uint64, _sz, _f32p]

    @staticmethod
    def _chk(st):
        if st != 0:
            raise OracleError(st)

    def generate_prototype(self, C_, T, beta=9.0, cutoff_scale=1.5):
        out = np.empty(C_ * T, np.float64)
        self._chk(self.lib.ppfo_generate_prototype(C_, T, beta, cutoff_scale, out))
        return out

    def fir(self, x, C_, T, coeffs, reference_order=False):
        x = _cf(x).reshape(-1)
        s_in = x.size // (2 * C_)
        out = np.empty(max(s_in - T + 1, 0) * C_ * 2, np.float32)
        self._chk(self.lib.ppfo_fir(x, s_in, C_, T, np.ascontiguousarray(coeffs, np.float64), out,
                                    int(reference_order)))
        return out

    def dft_naive(self, x):
        x = _cf(x).reshape(-1)
        out = np.empty_like(x)
        self._chk(self.lib.ppfo_dft_naive(x, x.size // 2, out))
        return out

    def fft(self, x):
        x = _cf(x).reshape(-1).copy()
        self._chk(self.lib.ppfo_fft(x, x.size // 2))
        return x

    def channelize(self, filt, C_, fft_fallback=True):
        filt = _cf(filt).reshape(-1)
        out = np.empty_like(filt)
        self._chk(self.lib.ppfo_channelize(filt, filt.size // (2 * C_), C_, int(fft_fallback), out))
        return out

    def fir_fft(self, x, C_, T, coeffs, fft_fallback=True):
        x = _cf(x).reshape(-1)
        s_in = x.size // (2 * C_)
        out = np.empty(max(s_in - T + 1, 0) * C_ * 2, np.float32)
        self._chk(self.lib.ppfo_fir_fft(x, s_in, C_, T, np.ascontiguousarray(coeffs, np.float64),
                                        int(fft_fallback), out))
        return out

    def mean_power(self, bins, C_):
        bins = _cf(bins).reshape(-1)
        out = np.empty(C_, np.float64)
        self._chk(self.lib.ppfo_mean_power(bins, bins.size // (2 * C_), C_, out))
        return out

    def process_stream(self, src: bytes, C_, T, block_spectra, coeffs, fft_fallback=True,
                       zero_prime=False):
        srcb = np.frombuffer(src, np.uint8) if len(src) else np.zeros(1, np.uint8)
        out = np.empty((len(src) // (8 * C_) + T + 1) * C_ * 8, np.uint8)
        st = StreamState()
        cf = np.ascontiguousarray(coeffs, np.float64)
        rc = self.lib.ppfo_process_stream(C_, T, block_spectra, int(fft_fallback),
                                          int(zero_prime), cf.ctypes.data, srcb, len(src), out,
                                          C.byref(st))
        if rc != 0:
            e = OracleError(rc)
            e.offset = st.error_offset
            raise e
        return out[: st.bytes_out].tobytes(), st

    def bessel_i0(self, x):
        st = C.c_int(0)
        v = self.lib.ppfo_bessel_i0(x, C.byref(st))
        self._chk(st.value)
        return v

    def flops_for_fir(self, c, t, s):
        return self.lib.ppfo_flops_for_fir(c, t, s)

    def synth(self, C_, n_samples, seed=1, first_sample=0):
        """The bench's synthetic tone + noise (same bytes as ppfg_synth)."""
        out = np.empty(2 * n_samples, np.float32)
        self._chk(self.lib.ppfo_synth(C_, seed, first_sample, n_samples, out))
        return out.view(np.complex64)

    def flops_for_dft(self, c, s):
        return self.lib.ppfo_flops_for_dft(c, s)


def _host_flags():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def ref_path():
    """Pick the reference build this host can execute: the -march=native one
    when this host has every ISA flag of the build host, else x86-64-v3."""
    native = os.path.join(_REF_DIR, "libppfref_native.so")
    v3 = os.path.join(_REF_DIR, "libppfref_v3.so")
    flags_file = os.path.join(_REF_DIR, "native_flags.txt")
    if os.path.exists(native) and os.path.exists(flags_file):
        need = {f for f in open(flags_file).read().split()
                if f.startswith(("avx", "fma", "bmi", "f16c", "amx", "sse", "vaes", "vpclmul",
                                 "gfni", "movbe", "adx", "sha"))}
        if need <= _host_flags():
            return native
    if os.path.exists(v3):
        return v3
    return None


class _Ref:
    def __init__(self, path):
        self.path = path
        L = self.lib = C.CDLL(path)
        L.ppfr_last_error.restype = C.c_char_p
        L.ppfr_generate_prototype.argtypes = [_sz, _sz, C.c_double, C.c_int, _f64p]
        L.ppfr_fir.argtypes = [_f32p, _sz, _sz, _sz, _f64p, _f32p, C.c_int, C.c_uint]
        L.ppfr_dft_naive.argtypes = [_f32p, _sz, _f32p]
        L.ppfr_fft.argtypes = [_f32p, _sz, _f32p]
        L.ppfr_channelize.argtypes = [_f32p, _sz, _sz, C.c_int, C.c_uint, _f32p]
        L.ppfr_fir_fft.argtypes = [_f32p, _sz, _sz, _sz, _f64p, C.c_int, C.c_uint, _f32p]
        L.ppfr_process_stream.argtypes = [_sz, _sz, _sz, C.c_int, C.c_int, C.c_void_p, _u8p, _sz,
                                          _u8p, C.POINTER(_sz), C.c_uint, C.POINTER(StreamState)]
        L.ppfr_compute_pass.argtypes = [_f32p, _sz, _sz, _sz, _f64p, _sz, C.c_uint, C.c_uint,
                                        _f64p, C.POINTER(C.c_uint64)]
        L.ppfr_bessel_i0.argtypes = [C.c_double, C.POINTER(C.c_int)]
        L.ppfr_bessel_i0.restype = C.c_double

    def _chk(self, st):
        if st != 0:
            raise OracleError(st, self.lib.ppfr_last_error().decode())

    def generate_prototype(self, C_, T, beta=9.0, rectangular=False):
        out = np.empty(C_ * T, np.float64)
        self._chk(self.lib.ppfr_generate_prototype(C_, T, beta, int(rectangular), out))
        return out

    def fir(self, x, C_, T, coeffs, reference=False, workers=1):
        x = _cf(x).reshape(-1)
        s_in = x.size // (2 * C_)
        out = np.empty(max(s_in - T + 1, 0) * C_ * 2, np.float32)
        self._chk(self.lib.ppfr_fir(x, s_in, C_, T, np.ascontiguousarray(coeffs, np.float64), out,
                                    int(reference), workers))
        return out

    def dft_naive(self, x):
        x = _cf(x).reshape(-1)
        out = np.empty_like(x)
        self._chk(self.lib.ppfr_dft_naive(x, x.size // 2, out))
        return out

    def fft(self, x):
        x = _cf(x).reshape(-1)
        out = np.empty_like(x)
        self._chk(self.lib.ppfr_fft(x, x.size // 2, out))
        return out

    def channelize(self, filt, C_, fft_fallback=True, workers=1):
        filt = _cf(filt).reshape(-1)
        out = np.empty_like(filt)
        self._chk(self.lib.ppfr_channelize(filt, filt.size // (2 * C_), C_, int(fft_fallback),
                                           workers, out))
        return out

    def fir_fft(self, x, C_, T, coeffs, fft_fallback=True, workers=1):
        x = _cf(x).reshape(-1)
        s_in = x.size // (2 * C_)
        out = np.empty(max(s_in - T + 1, 0) * C_ * 2, np.float32)
        self._chk(self.lib.ppfr_fir_fft(x, s_in, C_, T, np.ascontiguousarray(coeffs, np.float64),
                                        int(fft_fallback), workers, out))
        return out

    def process_stream(self, src: bytes, C_, T, block_spectra, coeffs=None, fft_fallback=True,
                       zero_prime=False, workers=1):
        srcb = np.frombuffer(src, np.uint8) if len(src) else np.zeros(1, np.uint8)
        out = np.empty((len(src) // (8 * C_) + T + 1) * C_ * 8, np.uint8)
        n = _sz(0)
        st = StreamState()
        cptr = None
        if coeffs is not None:
            cf = np.ascontiguousarray(coeffs, np.float64)
            cptr = cf.ctypes.data
        rc = self.lib.ppfr_process_stream(C_, T, block_spectra, int(fft_fallback),
                                          int(zero_prime), cptr, srcb, len(src), out, C.byref(n),
                                          workers, C.byref(st))
        if rc != 0:
            e = OracleError(rc, self.lib.ppfr_last_error().decode())
            e.offset = st.error_offset
            raise e
        return out[: n.value].tobytes(), st

    def compute_pass(self, x, C_, T, coeffs, block_spectra=4096, workers=1, reps=1):
        x = _cf(x).reshape(-1)
        secs = np.zeros(reps, np.float64)
        emitted = C.c_uint64(0)
        self._chk(self.lib.ppfr_compute_pass(x, x.size // (2 * C_), C_, T,
                                             np.ascontiguousarray(coeffs, np.float64),
                                             block_spectra, workers, reps, secs,
                                             C.byref(emitted)))
        return secs, emitted.value

    def bessel_i0(self, x):
        st = C.c_int(0)
        v = self.lib.ppfr_bessel_i0(x, C.byref(st))
        self._chk(st.value)
        return v


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def reference():
    """The compiled reference, or None where it was never built (GPU box
    without the traveling .so)."""
    global _ref
    if _ref is None:
        p = ref_path()
        if p is None and build_ref():
            p = ref_path()
        if p is None:
            return None
        _ref = _Ref(p)
    return _ref
