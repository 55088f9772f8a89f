// fused.cuh — K3: polyphase FIR + C-point FFT in one persistent kernel
// (channelize_block(ppf_fir_optimized(x)), pipeline.hpp:125-127), with no HBM
// round trip for the filtered block.
//
// Per CTA (one per SM): a contiguous range of output spectra, split into G
// groups (G > 1 only when C < 256*R so that every CTA still has 256 threads).
// Per group:
//   * TMA ring: P slots of one input spectrum each (N*8 bytes), filled by
//     1-D bulk copies (cp.async.bulk, SASS UBLKCP) on per-slot mbarriers; one
//     producer lane per group refills slots as soon as a batch has consumed
//     them, so HBM reads keep flowing while the CTA runs its FFT passes.
//   * FIR threads: thread j owns the R = 2^RLOG channels j + k*N/R. It keeps
//     their T-spectrum windows and taps in registers, slides them down the
//     time axis (each input read once from the ring), and for each output
//     spectrum immediately runs the first RLOG radix-2 stages on its R values
//     in registers (they pair exactly those channels: labels differing in the
//     top bits), then writes them to the FFT tile at the swizzled slots.
//   * FFT passes over the tile (B spectra per group per batch): the remaining
//     L - RLOG stages in register passes of <= W bits through shared memory;
//     the final pass stores natural-order bins straight to HBM, coalesced.
// EXACT = true accumulates the FIR in FP64 in the reference order (bit-exact
// to ppf_fir_optimized); false accumulates in FP32 (same order, one FMA per
// tap). The FFT is always the reference's exact radix-2 arithmetic.
#pragma once

#include <type_traits>

#include "fft.cuh"

namespace ppfg {

template <int L_, int T_, int RLOG_, bool EXACT_>
struct FusedCfg {
    static constexpr int L = L_, T = T_, RLOG = RLOG_;
    static constexpr bool EXACT = EXACT_;
    static constexpr int N = 1 << L;
    static constexpr int R = 1 << RLOG;
    static constexpr int NTG = N / R;                      // threads per group
    static constexpr int NT = NTG >= 256 ? NTG : 256;      // threads per CTA
    static constexpr int G = NT / NTG;                     // groups per CTA
    static constexpr int B = 8;                            // output spectra per group per batch
    static constexpr int P = 2 * B;                        // ring slots per group
    static constexpr int W = 4;                            // FFT pass width (16 values/thread)
    static constexpr unsigned STRIDE = sw_row_stride(N);
    // shared-memory layout (bytes)
    static constexpr size_t TW_BYTES = sizeof(float2) * ((N + 1) & ~1);
    static constexpr size_t RING_OFF = (TW_BYTES + 127) & ~size_t(127);
    static constexpr size_t RING_BYTES = sizeof(float2) * size_t(G) * P * N;
    static constexpr size_t TILE_OFF = RING_OFF + RING_BYTES;
    static constexpr size_t TILE_BYTES = sizeof(float2) * size_t(G) * B * STRIDE;
    static constexpr size_t BAR_OFF = (TILE_OFF + TILE_BYTES + 7) & ~size_t(7);
    static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) * G * P;
    static_assert(N % R == 0 && NT % NTG == 0, "bad fused shape");
};

// Output-row map for the final FFT pass: tile row r = g*B + i is output
// spectrum og0(g) + b*B + i of this CTA, if it exists.
struct FusedRows {
    long long o0, o1, rpg, base; // base = b*B
    int B;
    PPFG_DEV long long operator()(int r) const {
        const int g = r / B;
        const long long og0 = o0 + g * rpg;
        const long long og1 = min(og0 + rpg, o1);
        const long long s = og0 + base + (r - g * B);
        return s < og1 ? s : -1;
    }
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, 1)
    fused_fir_fft_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                         long long S_out, long long rows_per_cta, const float* __restrict__ taps,
                         const float2* __restrict__ tw_g) {
    constexpr int L = Cfg::L, T = Cfg::T, RLOG = Cfg::RLOG, N = Cfg::N, R = Cfg::R;
    constexpr int NTG = Cfg::NTG, NT = Cfg::NT, G = Cfg::G, B = Cfg::B, P = Cfg::P;
    using Acc = typename std::conditional<Cfg::EXACT, double, float>::type;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2* tw = reinterpret_cast<float2*>(smem_raw);
    float2* ring = reinterpret_cast<float2*>(smem_raw + Cfg::RING_OFF);
    float2* tile = reinterpret_cast<float2*>(smem_raw + Cfg::TILE_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + Cfg::BAR_OFF);

    const int tid = threadIdx.x;
    const int g = tid / NTG;
    const int j = tid - g * NTG;

    const long long o0 = static_cast<long long>(blockIdx.x) * rows_per_cta;
    const long long o1 = min(o0 + rows_per_cta, S_out);
    const long long rows_cta = max(o1 - o0, 0LL);
    const long long rpg = (rows_cta + G - 1) / G;
    const long long og0 = o0 + g * rpg;
    const long long og1 = min(og0 + rpg, o1);
    const long long n_out_g = max(og1 - og0, 0LL);
    const long long n_in_g = n_out_g > 0 ? n_out_g + T - 1 : 0;
    const float2* gsrc = in + og0 * N; // input spectrum q of the group = og0 + q
    float2* ring_g = ring + static_cast<size_t>(g) * P * N;
    uint64_t* bars_g = bars + g * P;

    for (int i = tid; i < N - 1; i += NT)
        tw[i] = tw_g[i];
    if (tid < G * P)
        mbar_init(bars + tid, 1);
    fence_mbar_init();
    __syncthreads();

    // ---- producer (lane j == 0 of each group) ----
    long long next_load = 0;
    auto issue = [&](long long q) {
        const int slot = static_cast<int>(q % P);
        mbar_arrive_expect_tx(bars_g + slot, N * sizeof(float2));
        bulk_g2s(ring_g + static_cast<size_t>(slot) * N, gsrc + q * N, N * sizeof(float2),
                 bars_g + slot);
    };
    if (j == 0) {
        for (; next_load < n_in_g && next_load < P; ++next_load)
            issue(next_load);
    }

    // ---- FIR state: taps and windows of channels c_k = j + k*NTG ----
    Acc h[R][T];
    Acc xr[R][T], xi[R][T];
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
            h[k][t] = static_cast<Acc>(__ldg(taps + static_cast<size_t>(t) * N + j + k * NTG));
            xr[k][t] = Acc(0);
            xi[k][t] = Acc(0);
        }
    }
    auto read_row = [&](long long q, float2 (&x)[R]) {
        const int slot = static_cast<int>(q % P);
        mbar_wait(bars_g + slot, static_cast<uint32_t>((q / P) & 1));
        const float2* row = ring_g + static_cast<size_t>(slot) * N + j;
#pragma unroll
        for (int k = 0; k < R; ++k)
            x[k] = row[k * NTG];
    };
    // warm-up: the first T-1 inputs fill window slots 1..T-1
#pragma unroll
    for (int q = 0; q + 1 < T; ++q) {
        float2 x[R];
        if (q < n_in_g) {
            read_row(q, x);
        } else {
#pragma unroll
            for (int k = 0; k < R; ++k)
                x[k] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
            xr[k][q + 1] = static_cast<Acc>(x[k].x);
            xi[k][q + 1] = static_cast<Acc>(x[k].y);
        }
    }
    __syncthreads();
    if (j == 0) {
        fence_proxy_async();
        for (; next_load < n_in_g && next_load < (T - 1) + P; ++next_load)
            issue(next_load);
    }

    const long long n_batches = (rpg + B - 1) / B;
    const unsigned swj = sw(static_cast<unsigned>(j));
    for (long long b = 0; b < n_batches; ++b) {
        // ---- FIR phase: B output spectra per group ----
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const long long rel = b * B + i;
            const bool valid = rel < n_out_g;
            float2 x[R];
            if (valid) {
                read_row(rel + T - 1, x);
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k)
                    x[k] = make_float2(0.f, 0.f);
            }
            float2 y[R];
#pragma unroll
            for (int k = 0; k < R; ++k) {
#pragma unroll
                for (int t = 0; t + 1 < T; ++t) {
                    xr[k][t] = xr[k][t + 1];
                    xi[k][t] = xi[k][t + 1];
                }
                xr[k][T - 1] = static_cast<Acc>(x[k].x);
                xi[k][T - 1] = static_cast<Acc>(x[k].y);
                Acc ar, ai;
                if constexpr (Cfg::EXACT) {
                    ar = __dmul_rn(h[k][0], xr[k][0]);
                    ai = __dmul_rn(h[k][0], xi[k][0]);
#pragma unroll
                    for (int t = 1; t < T; ++t) {
                        ar = __fma_rn(h[k][t], xr[k][t], ar);
                        ai = __fma_rn(h[k][t], xi[k][t], ai);
                    }
                    y[k] = make_float2(__double2float_rn(ar), __double2float_rn(ai));
                } else {
                    ar = __fmul_rn(h[k][0], xr[k][0]);
                    ai = __fmul_rn(h[k][0], xi[k][0]);
#pragma unroll
                    for (int t = 1; t < T; ++t) {
                        ar = __fmaf_rn(h[k][t], xr[k][t], ar);
                        ai = __fmaf_rn(h[k][t], xi[k][t], ai);
                    }
                    y[k] = make_float2(ar, ai);
                }
            }
            if constexpr (RLOG > 0)
                fft_stages<L, L - RLOG, RLOG, true>(y, static_cast<unsigned>(j), tw);
            float2* dst = tile + (g * B + i) * Cfg::STRIDE + swj;
#pragma unroll
            for (int k = 0; k < R; ++k)
                dst[sw(static_cast<unsigned>(k * NTG))] = y[k];
        }
        __syncthreads();
        // ---- refill the ring slots this batch consumed ----
        if (j == 0) {
            fence_proxy_async();
            const long long consumed = (b + 1) * B + T - 1; // inputs 0..consumed-1 read
            for (; next_load < n_in_g && next_load < consumed + P; ++next_load)
                issue(next_load);
        }
        // ---- remaining FFT stages, final pass stores to HBM ----
        FftPasses<L, L - RLOG, Cfg::W, false, true, NT>::run(
            nullptr, out, tile, Cfg::STRIDE, G * B, FusedRows{o0, o1, rpg, b * B, B}, tw);
        __syncthreads();
    }
}

} // namespace ppfg
