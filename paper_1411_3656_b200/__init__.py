"""paper_1411_3656_b200 — B200-native polyphase filter bank (arXiv 1411.3656).

The product is libppfg.so (paper_1411_3656_b200/csrc, C-ABI in include/ppfg.h)
with hand-written sm_100a kernels; `ppf` mirrors the reference's public API
over it. Importing this package does not touch the GPU; the first API call
loads (and if needed builds) the library and fails loudly if it cannot.
"""
from . import ppf  # noqa: F401
from .ppf import (EXACT, FAST, UNFUSED, FilterCoefficients, Plan, Stream,  # noqa: F401
                  channelize_block, dft_naive, fft, generate_prototype, ppf_fir_optimized,
                  ppf_fir_reference, process_stream, shard_range, synth)

__all__ = ["ppf", "Plan", "Stream", "FilterCoefficients", "generate_prototype",
           "ppf_fir_optimized", "ppf_fir_reference", "channelize_block", "fft", "dft_naive",
           "process_stream", "shard_range", "synth", "EXACT", "FAST", "UNFUSED"]
