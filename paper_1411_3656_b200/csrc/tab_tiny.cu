// tab_tiny.cu — K6 fused FIR + FFT for tiny power-of-two C (tiny.cuh):
// C = 1..32 at the acceptance tap counts T = 1, 2, 4, 8, 16 (FP32 and FP64
// FIR) and T = 32 (FP32; the FP64 window would not fit the registers).
#include "tables_impl.cuh"

namespace ppfg {

namespace {
template <int L, int T, bool EXACT>
KernelFn tiny() {
    return reinterpret_cast<KernelFn>(&fused_tiny_kernel<L, T, EXACT>);
}

template <int L>
KernelFn tiny_t(int T, bool exact) {
    switch (T) {
    case 1: return exact ? tiny<L, 1, true>() : tiny<L, 1, false>();
    case 2: return exact ? tiny<L, 2, true>() : tiny<L, 2, false>();
    case 4: return exact ? tiny<L, 4, true>() : tiny<L, 4, false>();
    case 8: return exact ? tiny<L, 8, true>() : tiny<L, 8, false>();
    case 16: return exact ? tiny<L, 16, true>() : tiny<L, 16, false>();
    case 32: return exact ? nullptr : tiny<L, 32, false>();
    default: return nullptr;
    }
}
} // namespace

KernelFn fir_c1_table(int T) {
    switch (T) {
    case 1: return reinterpret_cast<KernelFn>(&fir_c1_kernel<1>);
    case 2: return reinterpret_cast<KernelFn>(&fir_c1_kernel<2>);
    case 4: return reinterpret_cast<KernelFn>(&fir_c1_kernel<4>);
    case 8: return reinterpret_cast<KernelFn>(&fir_c1_kernel<8>);
    case 16: return reinterpret_cast<KernelFn>(&fir_c1_kernel<16>);
    case 32: return reinterpret_cast<KernelFn>(&fir_c1_kernel<32>);
    default: return nullptr;
    }
}

KernelFn tiny_table(int L, int T, bool exact) {
    switch (L) {
    case 0: return exact ? fir_c1_table(T) : nullptr; // C = 1: the coalesced FP64 FIR kernel
    case 1: return tiny_t<1>(T, exact);
    case 2: return tiny_t<2>(T, exact);
    case 3: return tiny_t<3>(T, exact);
    case 4: return tiny_t<4>(T, exact);
    case 5: return tiny_t<5>(T, exact);
    default: return nullptr;
    }
}

} // namespace ppfg
