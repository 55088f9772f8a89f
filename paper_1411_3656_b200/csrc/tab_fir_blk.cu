// tab_fir_blk.cu — K1b register-blocked FIR kernel instantiations.
#include "tables_impl.cuh"

namespace ppfg {

template <int T, int U, int NW, bool EXACT, int MINB, bool FFA = false>
FirBlkEntry fir_blk_entry() {
    using F = FirBlk<T, U, NW, EXACT>;
    return {reinterpret_cast<KernelFn>(&fir_block_kernel<T, U, NW, EXACT, MINB, FFA>), F::RB, F::NT,
            F::SMEM};
}

FirBlkEntry fir_blk_table(int T, bool exact) {
    if (exact) {
        switch (T) {
        case 16: return fir_blk_entry<16, 16, 4, true, 3>();
        case 20: return fir_blk_entry<20, 16, 4, true, 3>();
        case 24: return fir_blk_entry<24, 16, 4, true, 3>();
        case 32: return fir_blk_entry<32, 16, 4, true, 3>();
        case 48: return fir_blk_entry<48, 16, 4, true, 2>();
        case 64: return fir_blk_entry<64, 16, 4, true, 2>();
        default: return {};
        }
    }
    // FP32 (PPFG_FAST fir+fft only): the 2-parallel fast FIR (FFA, fir.cuh)
    // at T = 32 and 64 — 1 GiB fir+fft 0.443 -> 0.452 and 0.331 -> 0.344 of
    // roofline (U = 32 with 2 warps: 0.414 / 0.339)
    switch (T) {
    case 16: return fir_blk_entry<16, 16, 4, false, 3>();
    case 24: return fir_blk_entry<24, 16, 4, false, 3>();
    case 32: return fir_blk_entry<32, 16, 4, false, 3, true>();
    case 48: return fir_blk_entry<48, 16, 4, false, 3>();
    case 64: return fir_blk_entry<64, 16, 4, false, 3, true>();
    case 96: return fir_blk_entry<96, 16, 4, false, 2>();
    case 128: return fir_blk_entry<128, 16, 2, false, 3>();
    default: return {};
    }
}

} // namespace ppfg
