// tab_fir_blk.cu — K1b register-blocked FIR kernel instantiations.
#include "tables_impl.cuh"

namespace ppfg {

template <int T, int U, int NW, bool EXACT, int MINB>
FirBlkEntry fir_blk_entry() {
    using F = FirBlk<T, U, NW, EXACT>;
    return {reinterpret_cast<KernelFn>(&fir_block_kernel<T, U, NW, EXACT, MINB>), F::RB, F::NT,
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
    switch (T) {
    case 16: return fir_blk_entry<16, 16, 4, false, 3>();
    case 24: return fir_blk_entry<24, 16, 4, false, 3>();
    case 32: return fir_blk_entry<32, 16, 4, false, 3>();
    case 48: return fir_blk_entry<48, 16, 4, false, 3>();
    case 64: return fir_blk_entry<64, 16, 4, false, 3>();
    case 96: return fir_blk_entry<96, 16, 4, false, 2>();
    case 128: return fir_blk_entry<128, 16, 2, false, 3>();
    default: return {};
    }
}

} // namespace ppfg
