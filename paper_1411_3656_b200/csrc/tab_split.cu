// tab_split.cu — K3s split fused FIR+FFT kernels on thread-block clusters.
#include "tables_impl.cuh"

namespace ppfg {

std::vector<FusedEntry> fused_part_split() {
    // Round 2: per-pass-group owner-tile handoff (SplitCfg HS, the 11th
    // argument) where it measured faster (1 GiB): C=1024 T=16 0.645 -> 0.70,
    // EXACT C=1024 T=8 0.63 -> 0.645 (6.5 GB SKA EXACT 0.668 -> 0.682), EXACT
    // T=16 0.403 -> 0.411, C=2048 0.69 -> 0.71, C=4096 0.533 -> 0.537, T=32
    // 0.416 -> 0.420; not EXACT C=2048 (0.474 -> 0.463). Register splits with
    // HS (two A/B rounds): C=4096 FIR/FFT 168/88 0.537 -> 0.562; 128/128 and
    // 144/112 elsewhere, and flipping the float4 twiddles, all measured slower.
    // Paired FIR chains (SplitCfg PAIR, 12th argument) where they helped: EXACT
    // T=16 0.41 -> 0.428, EXACT C=2048 0.474 -> 0.481 (FAST T=16, C=2048 and
    // EXACT T=8 lost 1-4 %). Four FIR warpgroups with one channel per thread
    // (the TSPLIT input view): EXACT T=8 0.645 -> 0.53-0.54, FAST T=16 (W=4)
    // 0.70 -> 0.70 / (W=5) 0.55 — the smaller FFT role (80 registers) loses.
    // Trivial-twiddle prestages (SplitCfg TRIV, 13th argument, FAST): C=2048
    // 0.739 -> 0.751, C=4096 0.577 -> 0.596; C=1024 T=16 (one prestage) 0.72
    // either way.
    return {
        // thread-block clusters, FIR split by channel block and FFT by
        // spectrum (fused_split.cuh) — for FIR state that does not fit one SM.
        // preferred = taken by default: measured faster than FIR -> HBM -> FFT
        // (round 1, 1 GiB inputs: C=1024 T=16 0.62 vs 0.32 of HBM roofline,
        // T=32 0.41 vs 0.18, FP64 T=8 0.62 vs 0.42, FP64 T=16 0.40 vs 0.32,
        // C=2048 0.51 vs 0.42, FP64 C=2048 0.47 vs 0.42, C=4096 0.43 vs 0.38;
        // C=8192 0.29 vs 0.32 stays opt-in via PPFG_CLUSTER)
        // (float4 twiddle tables where they measured faster: FAST C=1024
        // T=16 0.62 vs 0.58, EXACT C=1024 T=16 0.40 vs 0.39, EXACT C=2048
        // 0.47 vs 0.44; FAST C=2048/4096 gained 15-27 % from float2)
        // (T=32 FAST: the unfused K1b FP32 FIR -> FFT measured 0.43 vs 0.42;
        // FIR/FFT registers 136/120 instead of 152/104 at FAST C=1024 T=16
        // 0.645 vs 0.619 and C=2048 0.688 vs 0.624 — not at C=4096 or FP64 C=2048;
        // FP64 C=1024 T=8 with float4 twiddles 0.629 vs 0.620 over four A/B
        // pairs; 4-CTA clusters 0.51, W=4 passes 0.44, FIR 168/88 0.44.
        // Rejected in the same A/B: FAST C=4096 float4 0.42 / 8-CTA 0.31 vs
        // 0.53; FP64 T=16 168/88 0.402 vs 0.403; FAST T=32 cluster 136/120
        // 0.41, 168/88 0.42, 8-CTA 0.28 — all below unfused K1b 0.43)

        split_entry<SplitCfg<10, 1, 16, false, 2, 5, 136, 120, 0, true, true>>(true),
        split_entry<SplitCfg<10, 2, 32, false, 2, 5, 152, 104, 0, true, true>>(false),
        split_entry<SplitCfg<10, 1, 8, true, 2, 5, 136, 120, 0, true, true>>(true),
        split_entry<SplitCfg<10, 2, 16, true, 2, 5, 152, 104, 0, true, true, true>>(true),
        split_entry<SplitCfg<11, 1, 8, false, 2, 5, 136, 120, 0, false, true, false, true>>(true),
        split_entry<SplitCfg<11, 2, 8, true, 2, 5, 152, 104, 0, true, false, true>>(true),
        split_entry<SplitCfg<12, 2, 8, false, 2, 5, 168, 88, 0, false, true, false, true>>(true),
        split_entry<SplitCfg<13, 3, 8, false>>(false),
    };
}

} // namespace ppfg
