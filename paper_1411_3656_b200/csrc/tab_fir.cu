// tab_fir.cu — K1 / K1t / K1f FIR kernel instantiations.
#include "tables_impl.cuh"

namespace ppfg {

template <int TC, int K>
FirEntry fir_entry() {
    constexpr int LAG = K == 1 ? 1 : (TC % 4 == 0 ? 4 : (TC % 2 == 0 ? 2 : 1));
    return {reinterpret_cast<KernelFn>(&fir_chain_kernel<TC, K, LAG>), TC, K};
}

template <int TC, int K, int RB, int MINB = 2>
FirTmaEntry fir_tma_entry() {
    constexpr int LAG = K == 1 ? 1 : (TC % 4 == 0 ? 4 : (TC % 2 == 0 ? 2 : 1));
    using F = FirTma<TC, K, LAG, RB>;
    return {reinterpret_cast<KernelFn>(&fir_tma_kernel<TC, K, LAG, RB, MINB>), K, RB, F::SMEM};
}

// K1t shapes (TMA-staged input; measured FIR-only at C = 1024: T = 8 0.87 vs
// 0.79, T = 16 0.66 vs 0.50, T = 32 (one lane per channel, 244 registers,
// 8 warps/SM) 0.36 vs 0.23 of the HBM roofline). Lane-chained K1t variants
// measured slower than the register-prefetch K1, which keeps the other T.
FirTmaEntry fir_tma_table(int T) {
    switch (T) {
    case 4: return fir_tma_entry<4, 1, 8>();
    case 8: return fir_tma_entry<8, 1, 8>();
    case 12: return fir_tma_entry<12, 1, 8>();
    case 16: return fir_tma_entry<16, 1, 8>();
    case 32: return fir_tma_entry<32, 1, 8, 1>();
    default: return {};
    }
}

template <int TC, int K, int RB>
FirTmaEntry fir_fast_entry() {
    return {reinterpret_cast<KernelFn>(&fir_fast_kernel<TC, K, RB>), K, RB, FirFast<TC, K, RB>::SMEM};
}

// K1f shapes: FP32 FIR for PPFG_FAST where no fused kernel covers T
FirTmaEntry fir_fast_table(int T) {
    switch (T) {
    case 32: return fir_fast_entry<16, 2, 8>();
    case 64: return fir_fast_entry<16, 4, 8>();
    case 128: return fir_fast_entry<16, 8, 8>();
    default: return {};
    }
}

// K1 variants: one lane per channel up to T = 16; larger T split over K
// lanes of up to 16 taps (T = TC * K), chained with a lag (fir.cuh).
FirEntry fir_table(int T) {
    switch (T) {
#define PPFG_FIR(t, tc, k)                                                                        \
    case t:                                                                                       \
        return fir_entry<tc, k>();
        PPFG_FIR(1, 1, 1) PPFG_FIR(2, 2, 1) PPFG_FIR(3, 3, 1) PPFG_FIR(4, 4, 1)
        PPFG_FIR(5, 5, 1) PPFG_FIR(6, 6, 1) PPFG_FIR(7, 7, 1) PPFG_FIR(8, 8, 1)
        PPFG_FIR(9, 9, 1) PPFG_FIR(10, 10, 1) PPFG_FIR(11, 11, 1) PPFG_FIR(12, 12, 1)
        PPFG_FIR(13, 13, 1) PPFG_FIR(14, 14, 1) PPFG_FIR(15, 15, 1) PPFG_FIR(16, 16, 1)
        PPFG_FIR(20, 10, 2) PPFG_FIR(24, 12, 2) PPFG_FIR(28, 14, 2) PPFG_FIR(32, 16, 2)
        PPFG_FIR(40, 10, 4) PPFG_FIR(48, 16, 3) PPFG_FIR(56, 14, 4) PPFG_FIR(64, 16, 4)
        PPFG_FIR(96, 16, 6) PPFG_FIR(128, 16, 8)
#undef PPFG_FIR
    default:
        return {nullptr, 0, 0};
    }
}

} // namespace ppfg
