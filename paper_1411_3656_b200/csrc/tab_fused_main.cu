// tab_fused_main.cu — K3 fused FIR+FFT shapes at T = 4, 8, 16 (C = 64..1024): the hot-path entries.
// Which (C, T) get a fused kernel: register budget per SM ~ C * (3T fp32 |
// 6T fp64) for the FIR windows + taps, plus the FFT pass registers. Entries
// with (120, 80, 2, 3) run three FFT warpgroups (640 threads): measured faster
// where the FFT role is critical (C=1024/T=8, C=64, T=1 at C<=128), slower
// elsewhere (round-1 sweep, profiles/round1/sweep.md).
#include "tables_impl.cuh"

namespace ppfg {

std::vector<FusedEntry> fused_part_main() {
    // Round 2: per-pass-group tile handoff (FusedCfg HS, the 12th argument)
    // wherever it applies (one FIR group, evenly split tile) and measured
    // faster (1 GiB, fraction of the measured HBM peak, two A/B rounds):
    // C=1024 T=8 FAST 0.81 -> 0.93 (6.5 GB SKA bench 0.868 -> 0.994; with the
    // trivial-twiddle prestages TRIV as well 1.001), C=1024 T=4 FAST (with
    // TRIV) 0.848 -> 0.856, EXACT 0.76 -> 0.80, C=512 T=16 0.755 -> 0.82,
    // EXACT C=512 T=8 0.68 -> 0.77, EXACT C=256 T=16 0.53 -> 0.56, C=256 T=32
    // 0.605 -> 0.635. Not on the T = 1 FFT entries (C=256 0.90 -> 0.85,
    // C=1024 0.884 -> 0.868) nor TRIV there (channelize_block must stay
    // bit-exact). With HS the SKA entry no longer gains from the L2 prefetch
    // one chunk ahead (L2A): 6.5 GB bench 3236-3242 with it, 3279-3283
    // without, 3105-3108 two chunks ahead. With several FIR groups per CTA (C <= 512 at R = 4,
    // C <= 256 at R = 2) HS helped every EXACT shape (C=128 T=8 0.71 -> 0.75,
    // C=256 0.756 -> 0.769, C=512 T=4 0.85 -> 0.90), FAST at T >= 16 (C=256
    // T=16 0.84 -> 0.86, C=128 T=32 0.626 -> 0.644), C=64 T=8 (0.88 -> 0.92)
    // and C=256 T=4 (0.794 -> 0.81), but not FAST C=128..512 at T=8 (cfg1
    // C=512: 0.90 -> 0.82) nor C=512 T=4 (0.89 -> 0.85): those keep
    // whole-tile handoff. Fewer channels per FIR thread (RLOG) make one FIR
    // group per CTA, where HS applies: C=512 T=8 (cfg1) R=2 + HS 0.90 -> 0.94,
    // C=256 T=8 R=1 + HS 0.82 -> 0.92 (R = 2 without HS: 0.89-0.925), C=128
    // T=8 R=2 + HS 0.866 -> 0.918, C=256 T=4 R=1 + HS 0.814 -> 0.878 (C=512
    // T=4 kept: 0.885 vs 0.865-0.883), C=128 T=16 R=1 0.763 -> 0.908, EXACT
    // C=128 T=8 R=1 0.745 -> 0.785, EXACT C=256 T=4 R=2 0.745 -> 0.905 (one
    // step fewer lost at C=64 T=4/8, C=128 T=4, EXACT C=256 T=8, C=512 T=4).
    // Late round 2: the one-stage trivial prestage (TRIV at R = 2) where it
    // measured faster: C=128 T=8 0.969 -> 0.975, C=512 T=16 0.857 -> 0.864
    // (cfg1 C=512 T=8 lost 0.6 %, C=64 even).
    // Late round 2: C=1024 T=4 FAST on three FFT warpgroups with float4
    // twiddles (the SKA entry's split) 0.888 -> 0.92-0.93; the same split
    // lost for EXACT C=512 T=8 (0.80 -> 0.71) and detection (0.448 -> 0.427).
    // Paired FIR chains (PAIR, 14th argument) on the EXACT shapes with one
    // channel per FIR thread: C=128 T=8 0.78 -> 0.83, C=256 T=16 0.556 -> 0.58
    // (FAST shapes and EXACT C=512 lost 1-4 %).
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
        fused_entry<FusedCfg<10, 8, 2, false, 120, 80, 2, 3, 2, true, 0, true, true>>(),
        // detection (mean power) at the SKA shape: two FFT warpgroups with 96
        // registers hold the per-bin accumulators next to the pass values
        power_entry<FusedCfg<10, 8, 2, false, 160, 96, 2, 2, 2, true, 0, true, true>>(),
        fused_entry<FusedCfg<9, 8, 1, false, 120, 80, 2, 3, 2, false, 0, true>>(),
        fused_entry<FusedCfg<8, 8, 0, false, 120, 80, 2, 3, 2, false, 0, true>>(),
        fused_entry<FusedCfg<7, 8, 1, false, 120, 80, 2, 3, 2, false, 0, true, true>>(),
        fused_entry<FusedCfg<6, 8, 1, false, 120, 80, 2, 3, 2, true, 0, true>>(),
        fused_entry<FusedCfg<10, 4, 2, false, 120, 80, 2, 3, 2, true, 0, true, true>>(),
        fused_entry<FusedCfg<9, 16, 1, false, 136, 120, 4, 2, 2, false, 0, true, true>>(),
        fused_entry<FusedCfg<9, 8, 1, true, 160, 96, 4, 2, 2, true, 0, true>>(),
        fused_entry<FusedCfg<8, 8, 1, true, 160, 96, 4, 2, 2, true, 0, true>>(),
        fused_entry<FusedCfg<7, 8, 0, true, 160, 96, 4, 2, 2, true, 0, true, false, true>>(),
        fused_entry<FusedCfg<6, 8, 1, true, 160, 96, 4, 2, 2, true, 0, true>>(),
        fused_entry<FusedCfg<10, 4, 2, true, 136, 120, 4, 2, 2, false, 0, true>>(),
    };
}

} // namespace ppfg
