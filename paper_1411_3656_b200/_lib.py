"""ctypes binding of libppfg.so (include/ppfg.h). Loading fails loudly: there
is no CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib = None

u64 = C.c_uint64
vp = C.c_void_p
dp = C.POINTER(C.c_double)

READ_FN = C.CFUNCTYPE(C.c_int64, vp, vp, u64)
WRITE_FN = C.CFUNCTYPE(C.c_int, vp, vp, u64)


class StreamState(C.Structure):
    _fields_ = [("spectra_processed", u64), ("bytes_in", u64), ("bytes_out", u64),
                ("dropped_samples", u64)]


# name -> (restype, argtypes); every symbol include/ppfg.h declares
SIGNATURES = {
    "ppfg_plan_create": (C.c_int, [C.POINTER(vp), u64, u64, dp, C.c_uint32, C.c_int]),
    "ppfg_plan_destroy": (C.c_int, [vp]),
    "ppfg_plan_stream": (vp, [vp]),
    "ppfg_fir": (C.c_int, [vp, vp, u64, vp, C.c_int, vp]),
    "ppfg_fir_reference_order": (C.c_int, [vp, vp, u64, vp, C.c_int, vp]),
    "ppfg_channelize": (C.c_int, [vp, vp, u64, vp, C.c_int, C.c_int, vp]),
    "ppfg_fir_fft": (C.c_int, [vp, vp, u64, vp, C.c_int, vp]),
    "ppfg_mean_power": (C.c_int, [vp, vp, u64, vp, C.c_int, vp]),
    "ppfg_fir_fft_mean_power": (C.c_int, [vp, vp, u64, vp, C.c_int, vp]),
    "ppfg_fir_fft_kind": (C.c_int, [vp]),
    "ppfg_fir_fft_kernel_name": (C.c_char_p, [vp]),
    "ppfg_device_hbm_gbs": (C.c_int, [C.c_int, dp]),
    "ppfg_host_copy": (C.c_int, [vp, vp, u64]),
    "ppfg_current_device": (C.c_int, [C.POINTER(C.c_int)]),
    "ppfg_fft": (C.c_int, [vp, u64, vp]),
    "ppfg_dft_naive": (C.c_int, [vp, u64, vp]),
    "ppfg_stream_open": (C.c_int, [C.POINTER(vp), vp, u64, C.c_int, C.c_int]),
    "ppfg_stream_push": (C.c_int, [vp, vp, u64, vp, u64, C.POINTER(u64)]),
    "ppfg_stream_close": (C.c_int, [vp, C.POINTER(StreamState)]),
    "ppfg_stream_destroy": (C.c_int, [vp]),
    "ppfg_process_stream": (C.c_int, [vp, u64, C.c_int, C.c_int, READ_FN, vp, WRITE_FN, vp,
                                      C.POINTER(StreamState)]),
    "ppfg_shard_range": (C.c_int, [u64, u64, C.c_int, C.c_int, C.POINTER(u64), C.POINTER(u64),
                                   C.POINTER(u64), C.POINTER(u64)]),
    "ppfg_multi_fir_fft": (C.c_int, [u64, u64, dp, C.c_uint32, C.POINTER(C.c_int), C.c_int, vp,
                                     u64, vp]),
    "ppfg_multi_fir_fft_device": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(u64),
                                            C.POINTER(vp), C.POINTER(u64)]),
    "ppfg_synth": (C.c_int, [u64, u64, u64, u64, vp, C.c_int, C.c_int, vp]),
    "ppfg_generate_prototype": (C.c_int, [u64, u64, C.c_double, C.c_double, dp]),
    "ppfg_flops_for_fir": (u64, [u64, u64, u64]),
    "ppfg_flops_for_dft": (u64, [u64, u64]),
    "ppfg_device_alloc": (C.c_int, [C.POINTER(vp), u64, C.c_int]),
    "ppfg_device_free": (C.c_int, [vp]),
    "ppfg_memcpy": (C.c_int, [vp, vp, u64]),
    "ppfg_plan_synchronize": (C.c_int, [vp]),
    "ppfg_last_error": (C.c_char_p, []),
    "ppfg_last_error_offset": (u64, []),
    "ppfg_kernel_launches": (u64, []),
    "ppfg_version": (C.c_char_p, []),
}


def so_path() -> str:
    return _build.SO


def load(build_if_needed: bool = True):
    """Load libppfg.so (building it with nvcc first if it is missing or stale).
    Raises OSError/CalledProcessError if that is impossible — never falls back."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        so = os.environ.get("PPFG_SO")  # A/B experiments with another build of the library
        if so is None:
            if build_if_needed and _build.stale():
                _build.build()
            so = _build.SO
        if not os.path.exists(so):
            raise OSError(f"libppfg.so not found at {so}; run __graft_entry__.build()")
        lib = C.CDLL(so)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        if hasattr(lib, "ppfg_debug_trace"):  # -DPPFG_TRACE debug builds only
            lib.ppfg_debug_trace.argtypes = [vp]
        _lib = lib
        return lib
