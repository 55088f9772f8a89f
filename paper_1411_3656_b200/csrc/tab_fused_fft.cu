// tab_fused_fft.cu — K3 with T = 1: fir+fft plans with a single tap (channelize_block itself
// takes the K2n tile FFT since late round 2).
#include "tables_impl.cuh"

namespace ppfg {

std::vector<FusedEntry> fused_part_fft() {
    return {
        // T = 1: x*h with one tap, then the bit-exact FFT; until late round 2
        // also channelize_block (unit taps) for 64 <= C <= 4096
        // (C = 4096: 0.76 of roofline vs 0.69 for K2)
        // (split-kernel T = 1 entries for C = 4096, 8192 and FP64 C = 4096 on
        // 8-CTA clusters measured slower than K2 / the unfused path)
        // (round 2, C = 64..1024: three FFT warpgroups, float4 twiddles and
        // the per-pass-group handoff, as the T = 8 entries — 1 GiB back to
        // back: C=64 0.850 -> 0.878, C=1024 0.914 -> 0.919-0.929; without the
        // handoff C=256/512 lost 8 %)
        fused_entry<FusedCfg<6, 1, 0, false, 120, 80, 2, 3, 2, true, 0, true>>(),
        fused_entry<FusedCfg<7, 1, 0, false, 120, 80, 2, 3, 2, true, 0, true>>(),
        fused_entry<FusedCfg<8, 1, 0, false, 120, 80, 2, 3, 2, true, 0, true>>(),
        fused_entry<FusedCfg<9, 1, 1, false, 120, 80, 2, 3, 2, true, 0, true>>(),
        fused_entry<FusedCfg<10, 1, 2, false, 120, 80, 2, 3, 2, true, 0, true>>(),
        fused_entry<FusedCfg<11, 1, 3, false, 160, 96, 3>>(),
        fused_entry<FusedCfg<12, 1, 4, false, 160, 96, 2>>(),
    };
}

} // namespace ppfg
