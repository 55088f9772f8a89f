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

FftEntry fft_ring_entry() {
    using F = FftRing<13, kFftW, kRingNT>;
    return {reinterpret_cast<KernelFn>(&fft_ring_kernel<13, kFftW, kRingNT>), F::SMEM, F::NT, 1};
}

} // namespace ppfg
