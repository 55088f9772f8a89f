// tab_fft.cu — K2 row FFT and K2n tile FFT instantiations.
#include "tables_impl.cuh"

namespace ppfg {

template <int L>
FftEntry fft_entry() {
    constexpr bool tws = L <= 11;
    constexpr int rb = (kFftNT << kFftW) / (1 << L) > 0 ? (kFftNT << kFftW) / (1 << L) : 1;
    return {reinterpret_cast<KernelFn>(&fft_rows_kernel<L, kFftW, tws, kFftNT>),
            fft_rows_smem_bytes<L, kFftW, tws, kFftNT>(), kFftNT, rb};
}

const FftEntry* fft_table(int L) {
    static const FftEntry t[kFftMaxL + 1] = {
        {nullptr, 0, 0, 0},  fft_entry<1>(),  fft_entry<2>(),  fft_entry<3>(),  fft_entry<4>(),
        fft_entry<5>(),      fft_entry<6>(),  fft_entry<7>(),  fft_entry<8>(),  fft_entry<9>(),
        fft_entry<10>(),     fft_entry<11>(), fft_entry<12>(), fft_entry<13>(),
    };
    if (L < 1 || L > kFftMaxL)
        return nullptr;
    return &t[L];
}

template <int L, int NT, int MINB = 1, int W = kFftW, int UPT = 1, bool VOLTW = false,
          bool TWL = false>
FftEntry fft_tiles_one() {
    using F = FftTiles<L, W, NT, UPT, TWL>;
    return {reinterpret_cast<KernelFn>(&fft_tiles_kernel<L, W, NT, MINB, UPT, VOLTW, TWL>), F::SMEM,
            NT, F::NR};
}

// Per C the (threads, units per thread, pass width) that measured fastest
// (1 GiB back to back, fraction of the measured HBM peak; the kernel it
// replaced in brackets — K3 with T = 1, at C = 8192 the persistent TMA-ring
// K2r; cuFFT after the slash):
//   C=64 1.03 (0.88) / 0.99    C=128 1.04 (0.94) / 1.04   C=256 1.04 (0.94) / 1.05
//   C=512 1.04 (0.95) / 1.04   C=1024 1.01 (0.92) / 1.04  C=2048 0.97 (0.88) / 0.97
//   C=4096 0.95 (0.86) / 0.92  C=8192 0.84 (0.76) / 0.80
// C=1024 reads its twiddles with volatile shared loads (TwV2): with ordinary
// loads its 5-bit passes are hoisted into 198 registers (0.80); 4-bit passes
// 0.935. From C=2048 the tiles keep only the first passes' twiddles in shared
// memory (TWL: 2-4 KB instead of 16-64 KB) and the last pass reads the table
// from global (its lanes read consecutive entries). Rejected per C: 512-thread
// tiles (0.54-0.60), 16 KB tiles at C=64/256 (0.80-0.81), 6-bit passes at
// C=2048 (0.80-0.92), twiddles of every pass from global (0.38-0.63).
FftEntry fft_tiles_entry(int L) {
    switch (L) {
    case 6: return fft_tiles_one<6, 128, 1, kFftW, 4>();   // 64 rows (32 KB) per CTA
    case 7: return fft_tiles_one<7, 256>();                // 32 rows
    case 8: return fft_tiles_one<8, 128, 1, kFftW, 2>();   // 16 rows
    case 9: return fft_tiles_one<9, 128>();                // 8 rows
    case 10: return fft_tiles_one<10, 128, 1, kFftW, 1, true>(); // 4 rows, volatile twiddle loads
    // C >= 2048: only the first passes' twiddles in shared memory, the last
    // pass reads the table from global (TWL)
    case 11: return fft_tiles_one<11, 128, 1, kFftW, 2, false, true>(); // 2 rows
    case 12: return fft_tiles_one<12, 128, 1, kFftW, 2, false, true>(); // 1 row
    case 13: return fft_tiles_one<13, 128, 1, kFftW, 2, false, true>(); // 1 row (64 KB)
    default: return {};
    }
}

} // namespace ppfg
