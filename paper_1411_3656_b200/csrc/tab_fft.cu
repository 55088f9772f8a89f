// tab_fft.cu — K2 row FFT and K2r TMA-ring FFT instantiations.
#include "tables_impl.cuh"

namespace ppfg {

constexpr int kRingNT = 0; // K2r threads per CTA (0: one first-pass unit per thread; 512 measured the same)

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

template <int L, int NT, int MINB = 1, int W = kFftW, int UPT = 1, bool VOLTW = false>
FftEntry fft_tiles_one() {
    using F = FftTiles<L, W, NT, UPT>;
    return {reinterpret_cast<KernelFn>(&fft_tiles_kernel<L, W, NT, MINB, UPT, VOLTW>), F::SMEM, NT,
            F::NR};
}

// Per C the (threads, units per thread, pass width) that measured fastest
// (1 GiB back to back, fraction of the measured HBM peak; the earlier
// channelize_block kernel K3(T=1) in brackets; cuFFT after the slash):
// C=64 1.03 (0.88) / 0.99, C=128 1.04 (0.94) / 1.04, C=256 1.04 (0.94) / 1.05,
// C=512 1.04 (0.95) / 1.04, C=1024 1.01 (0.92) / 1.04, C=2048 0.91 (0.88) / 0.97.
// At C=4096 the K3(T=1) kernel stays (0.86 vs 0.81-0.86). C=1024 needs the
// volatile twiddle loads (TwV2): with ordinary loads its 5-bit passes take
// 198 registers (0.80), 4-bit passes 0.935. Rejected per C: 512-thread tiles
// (0.54-0.60), 16 KB tiles at C=64/256 (0.80-0.81), 6-bit passes at C=2048
// (0.80-0.92).
FftEntry fft_tiles_entry(int L) {
    switch (L) {
    case 6: return fft_tiles_one<6, 128, 1, kFftW, 4>();   // 64 rows (32 KB) per CTA
    case 7: return fft_tiles_one<7, 256>();                // 32 rows
    case 8: return fft_tiles_one<8, 128, 1, kFftW, 2>();   // 16 rows
    case 9: return fft_tiles_one<9, 128>();                // 8 rows
    case 10: return fft_tiles_one<10, 128, 1, kFftW, 1, true>(); // 4 rows, volatile twiddle loads
    case 11: return fft_tiles_one<11, 256, 1, kFftW, 2>(); // 4 rows (64 KB)
    case 12: return {}; // K3(T=1)
    default: return {};
    }
}

FftEntry fft_ring_entry() {
    using F = FftRing<13, kFftW, kRingNT>;
    return {reinterpret_cast<KernelFn>(&fft_ring_kernel<13, kFftW, kRingNT>), F::SMEM, F::NT, 1};
}

} // namespace ppfg
