// fir.cuh — K1: the polyphase FIR stage, bit-exact to ppf_fir_optimized.
//
// Reference contract (fir.hpp:85-110, 158-212): y[s][c] = sum_t h[t][c] x[s+t][c]
// over valid windows, each output component accumulated in double as
// acc = h0*x0 (a product), then acc = fma(h_t, x_t, acc) for t = 1..T-1 in
// ascending order, then rounded to float. Taps are the f32-quantised values.
// Products of two floats are exact in double, so DFMA on the same operands in
// the same order reproduces every bit; fma(h0, x0, -0.0) == h0*x0 including
// the sign of zero, and fma(h0, x0, +0.0) is ppf_fir_reference's start.
//
// Mapping (fir_chain_kernel<TC, K>): T = TC*K taps are split over K lanes of
// a warp. Lane q owns taps [q*TC, (q+1)*TC) of one channel and slides a
// TC-spectrum window (doubles: each input converted once) down its time
// segment. The accumulator of output s visits lane 0 at step s, lane 1 at
// step s+1, ... (a shuffle per step), so every output still sees its taps in
// ascending order, one DFMA after another, while per-lane registers stay at
// 6*TC. K = 1 (T <= 16) is the plain one-channel-per-lane kernel. Lanes of a
// chunk take consecutive channels, so loads/stores coalesce; the step loop is
// unrolled by TC so the window is a circular register file (no moves).
#pragma once

#include "common.cuh"

namespace ppfg {

template <int TC, int K, int LAG>
__global__ void __launch_bounds__(256) fir_chain_kernel(const float2* __restrict__ in,
                                                        float2* __restrict__ out, unsigned C,
                                                        long long S_in, long long S_out,
                                                        const float* __restrict__ taps, int seg,
                                                        long long n_tasks, double init) {
    constexpr int CPW = 32 / K; // channels per warp
    const int lane = threadIdx.x & 31;
    const int q = lane / CPW;   // tap chunk of this lane (q >= K: idle lane)
    const int cl = lane - q * CPW;
    const long long task = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (task >= n_tasks)
        return;
    const long long n_cb = (C + CPW - 1) / CPW;
    const long long sg = task / n_cb;
    const unsigned c_raw = static_cast<unsigned>((task - sg * n_cb) * CPW + cl);
    const bool live = q < K && c_raw < C;
    const unsigned c = live ? c_raw : 0u;
    const int qq = q < K ? q : K - 1;
    const long long s0 = sg * seg;
    const long long s1 = min(s0 + seg, S_out);
    const int steps = static_cast<int>(s1 - s0) + LAG * (K - 1);

    double h[TC];
#pragma unroll
    for (int t = 0; t < TC; ++t)
        h[t] = static_cast<double>(__ldg(taps + static_cast<size_t>(qq * TC + t) * C + c));

    // lane q at step tau computes output s = s0 + tau - LAG*q over inputs
    // s + q*TC + [0, TC); its accumulator arrives from lane q-1, which ran
    // that output LAG steps earlier, so LAG consecutive steps' DFMA chains are
    // independent and overlap. Per step the lane loads input
    // s0 + tau + q*(TC-LAG) + TC-1. Indices are clamped into [0, S_in): clamped
    // loads only feed outputs outside [s0, s1), which are never stored.
    static_assert(TC % LAG == 0, "LAG must divide TC");
    const long long base = s0 + static_cast<long long>(qq) * (TC - LAG);
    auto ld = [&](long long idx) {
        idx = min(max(idx, 0LL), S_in - 1);
        return __ldcs(in + idx * C + c);
    };
    double2 w[TC];
#pragma unroll
    for (int t = 0; t + 1 < TC; ++t) {
        const float2 x = ld(base + t);
        w[t] = make_double2(x.x, x.y);
    }
    const unsigned src_lane_off = CPW;
    double2 carry[LAG];
#pragma unroll
    for (int i = 0; i < LAG; ++i)
        carry[i] = make_double2(0.0, 0.0);
    // software pipeline: the TC inputs of the next block are in flight while
    // the current block computes (TC loads per warp always outstanding)
    float2 nx[TC];
#pragma unroll
    for (int u = 0; u < TC; ++u)
        nx[u] = ld(base + u + TC - 1);
    for (int tau0 = 0; tau0 < steps; tau0 += TC) {
        float2 cur[TC];
#pragma unroll
        for (int u = 0; u < TC; ++u) {
            cur[u] = nx[u];
            nx[u] = ld(base + tau0 + TC + u + TC - 1);
        }
#pragma unroll
        for (int u = 0; u < TC; ++u) {
            const int tau = tau0 + u;
            // newest input of this step goes to circular slot (u + TC - 1) % TC
            w[(u + TC - 1) % TC] = make_double2(cur[u].x, cur[u].y);
            // accumulator from the previous lane (its previous step)
            double2 acc = make_double2(init, init);
            if constexpr (K > 1) {
                acc.x = __shfl_up_sync(0xffffffffu, carry[u % LAG].x, src_lane_off);
                acc.y = __shfl_up_sync(0xffffffffu, carry[u % LAG].y, src_lane_off);
                if (qq == 0) {
                    acc.x = init;
                    acc.y = init;
                }
            }
#pragma unroll
            for (int t = 0; t < TC; ++t) {
                const double2 v = w[(u + t) % TC];
                acc.x = __fma_rn(h[t], v.x, acc.x);
                acc.y = __fma_rn(h[t], v.y, acc.y);
            }
            carry[u % LAG] = acc;
            const long long s = s0 + tau - static_cast<long long>(LAG) * qq;
            if (live && qq == K - 1 && q < K && tau < steps && s >= s0 && s < s1)
                __stcs(out + s * C + c, make_float2(__double2float_rn(acc.x),
                                                    __double2float_rn(acc.y)));
        }
    }
}

// Any T: the same op sequence, window re-read through L1/L2 per tap.
__global__ void __launch_bounds__(256) fir_exact_generic_kernel(const float2* __restrict__ in,
                                                                float2* __restrict__ out,
                                                                unsigned C, unsigned T,
                                                                long long S_out,
                                                                const float* __restrict__ taps,
                                                                int seg, long long n_work,
                                                                double init) {
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= n_work)
        return;
    const unsigned c = static_cast<unsigned>(g % C);
    const long long s0 = (g / C) * seg;
    const long long s1 = min(s0 + seg, S_out);
    for (long long s = s0; s < s1; ++s) {
        const float2* src = in + s * C + c;
        const double h0 = __ldg(taps + c);
        const float2 x0 = __ldg(src);
        double ar = __fma_rn(h0, static_cast<double>(x0.x), init);
        double ai = __fma_rn(h0, static_cast<double>(x0.y), init);
        for (unsigned t = 1; t < T; ++t) {
            const double ht = __ldg(taps + static_cast<size_t>(t) * C + c);
            const float2 x = __ldg(src + static_cast<long long>(t) * C);
            ar = __fma_rn(ht, static_cast<double>(x.x), ar);
            ai = __fma_rn(ht, static_cast<double>(x.y), ai);
        }
        out[s * C + c] = make_float2(__double2float_rn(ar), __double2float_rn(ai));
    }
}

} // namespace ppfg
