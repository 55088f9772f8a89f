// tab_fused_main.cu — K3 fused FIR+FFT shapes at T = 4, 8, 16 (C = 64..1024): the hot-path entries.
// Which (C, T) get a fused kernel: register budget per SM ~ C * (3T fp32 |
// 6T fp64) for the FIR windows + taps, plus the FFT pass registers. Entries
// with (120, 80, 2, 3) run three FFT warpgroups (640 threads): measured faster
// where the FFT role is critical (C=1024/T=8, C=64, T=1 at C<=128), slower
// elsewhere (round-1 sweep, profiles/round1/sweep.md).
#include "tables_impl.cuh"

namespace ppfg {

std::vector<FusedEntry> fused_part_main() {
    return {
        // (float4 twiddle tables where they measured faster than float2:
        // C=1024 T=8 FAST 0.86 vs 0.85 at the SKA size, C=512 EXACT 0.68 vs
        // 0.65, C=64 0.88 vs 0.86, EXACT C=64..256 +2-3 %; L2 prefetch one
        // chunk ahead at the SKA shape: 2836 vs 2802 GB/s on the 6.5 GB
        // bench (flat at 1 GiB; -1..2 % on other shapes); three FFT
        // warpgroups at C=128 0.87 vs 0.78, C=256 0.82 vs 0.76, C=512 0.91 vs
        // 0.90 — but not at C=1024 T=4: 0.83 vs 0.86; FIR/FFT registers
        // 136/120 instead of 160/96 at C=512 T=16 0.76 vs 0.72 and FP64
        // C=1024 T=4 0.762 vs 0.753)
        fused_entry<FusedCfg<10, 8, 2, false, 120, 80, 2, 3, 2, true, 1>>(),
        fused_entry<FusedCfg<9, 8, 2, false, 120, 80, 2, 3>>(),
        fused_entry<FusedCfg<8, 8, 2, false, 120, 80, 2, 3>>(),
        fused_entry<FusedCfg<7, 8, 2, false, 120, 80, 2, 3>>(),
        fused_entry<FusedCfg<6, 8, 1, false, 120, 80, 2, 3, 2, true>>(),
        fused_entry<FusedCfg<10, 4, 2, false>>(),
        fused_entry<FusedCfg<9, 16, 1, false, 136, 120>>(),
        fused_entry<FusedCfg<9, 8, 1, true, 160, 96, 4, 2, 2, true>>(),
        fused_entry<FusedCfg<8, 8, 1, true, 160, 96, 4, 2, 2, true>>(),
        fused_entry<FusedCfg<7, 8, 1, true, 160, 96, 4, 2, 2, true>>(),
        fused_entry<FusedCfg<6, 8, 1, true, 160, 96, 4, 2, 2, true>>(),
        fused_entry<FusedCfg<10, 4, 2, true, 136, 120>>(),
    };
}

} // namespace ppfg
