// tiny.cuh — K6: fused FIR + C-point FFT for small power-of-two channel
// counts (C = 1..32, SURVEY §8f row 2 "tiny C"), one warp-level kernel with
// no HBM round trip for the filtered block and no shared memory (C = 1: 32
// single-lane groups per warp, the 1-point FFT being the identity).
//
// A warp holds 32 / C lane groups; lane c of a group owns channel c of a
// contiguous time segment of output spectra. Per output spectrum the lane
//   - slides its channel's T-spectrum window down the time axis (registers,
//     circular by loop unrolling: every input sample is loaded once), and
//     filters it exactly as ppf_fir_optimized (fir.hpp:85-110): FP64 FMA in
//     ascending tap order from h0*x0 (EXACT) or an FP32 FFMA2 chain (FAST);
//   - runs the C-point radix-2 DIT FFT ACROSS the group's lanes: stage s pairs
//     the lanes whose labels (= channel indices, dft.hpp:106-112 bit
//     reversal folded into the labels, fft.cuh) differ in bit L - s; both
//     lanes of a pair get the partner's value by one shuffle and compute the
//     same t = w * hi with the reference's operations (dft.hpp:122-131), the
//     low lane keeping lo + t and the high lane lo - t: bit-identical to
//     FftPlan::transform;
//   - after the last stage lane c holds bin rev_L(c) and stores it: the group
//     writes its C-bin row as one contiguous (permuted) segment.
// Inputs are read through a register prefetch queue: the load of step
// tau + PF (8 or 16) is issued at step tau, so that many rows per lane are in
// flight while the window filters.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ppfg {

template <int L, int T, bool EXACT>
__global__ void __launch_bounds__(256) fused_tiny_kernel(const float2* __restrict__ in,
                                                         float2* __restrict__ out, long long S_in,
                                                         long long S_out, const float* __restrict__ taps,
                                                         const float2* __restrict__ tw, int seg,
                                                         long long n_tasks) {
    constexpr int N = 1 << L;   // channels (lanes per group)
    constexpr int G = 32 / N;   // groups (time segments) per warp
    static_assert(L >= 0 && L <= 5, "C = 1..32 (C = 1: the 1-point FFT is the identity)");
    using Acc = typename std::conditional<EXACT, double, float>::type;
    const int lane = threadIdx.x & 31;
    const int q = lane >> L;
    const int c = lane & (N - 1);
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (warp * G >= n_tasks) // whole warp idle (uniform: shuffles need the full warp)
        return;
    const long long task = warp * G + q;
    // a group past the last task runs the same (uniform) loop on row 0 and stores nothing
    const long long s0 = task < n_tasks ? task * seg : 0;
    const long long s1 = task < n_tasks ? min(s0 + seg, S_out) : 0;

    Acc h[T];
#pragma unroll
    for (int t = 0; t < T; ++t)
        h[t] = static_cast<Acc>(__ldg(taps + t * N + c));
    // this lane's twiddle per stage (the pair's shared tw[h-1+j], j from the
    // label bits above the stage's bit)
    float2 w[L > 0 ? L : 1];
#pragma unroll
    for (int s = 1; s <= L; ++s) {
        const int b = L - s;
        const unsigned j = s > 1 ? crev(static_cast<unsigned>(c) >> (b + 1), s - 1) : 0u;
        w[s - 1] = __ldg(tw + (1 << (s - 1)) - 1 + j);
    }
    const unsigned bin = crev(static_cast<unsigned>(c), L);

    auto ld = [&](long long row) {
        row = min(row, S_in - 1);  // past the end: only feeds outputs never stored
        return __ldcs(in + row * N + c);
    };
    using Win = typename std::conditional<EXACT, double2, float2>::type;
    Win xw[T];
#pragma unroll
    for (int t = 0; t + 1 < T; ++t) {
        const float2 x = ld(s0 + t);
        xw[t].x = x.x;
        xw[t].y = x.y;
    }
    // prefetch queue: the input of step tau + PF is loaded at step tau (16
    // rows in flight per lane; 8 at T = 32, where the window is large); the
    // step loop is unrolled by UNR = max(T, PF) so both the window slot and
    // the queue slot are compile-time
    // (measured at 1 GiB: 16 rows ahead helped every T = 16 shape and T = 8 at
    // C <= 8 or in FP64 — C=8 T=8 FP64 0.58 -> 0.70, C=16 T=16 0.57 -> 0.63 —
    // but not C=32 T=8 FP32 (0.735 -> 0.69) nor C=2 T=4 FP64 (0.51 -> 0.44))
    constexpr int PF = (T == 16 || (T == 8 && (EXACT || L <= 3))) ? 16 : 8;
    constexpr int UNR = T > PF ? T : PF;
    static_assert(UNR % T == 0 && UNR % PF == 0, "window and queue cycles divide the unroll");
    float2 nx[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u)
        nx[u] = ld(s0 + T - 1 + u);

    for (int tau0 = 0; tau0 < seg; tau0 += UNR) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            // newest input of this step -> circular slot (u + T - 1) % T
            const float2 x = nx[u % PF];
            nx[u % PF] = ld(s0 + tau0 + u + PF + T - 1);
            xw[(u + T - 1) % T].x = x.x;
            xw[(u + T - 1) % T].y = x.y;
            float2 y;
            if constexpr (EXACT) {
                double ar = __dmul_rn(h[0], xw[u % T].x);
                double ai = __dmul_rn(h[0], xw[u % T].y);
#pragma unroll
                for (int t = 1; t < T; ++t) {
                    ar = __fma_rn(h[t], xw[(u + t) % T].x, ar);
                    ai = __fma_rn(h[t], xw[(u + t) % T].y, ai);
                }
                y = make_float2(__double2float_rn(ar), __double2float_rn(ai));
            } else {
                y = mul2s(h[0], xw[u % T]);
#pragma unroll
                for (int t = 1; t < T; ++t)
                    y = fma2s(h[t], xw[(u + t) % T], y);
            }
            // C-point FFT across the group's lanes (labels = lane channel c)
#pragma unroll
            for (int s = 1; s <= L; ++s) {
                const int b = L - s;
                const bool upper = (c >> b) & 1;
                const float px = __shfl_xor_sync(0xffffffffu, y.x, 1 << b);
                const float py = __shfl_xor_sync(0xffffffffu, y.y, 1 << b);
                const float lx = upper ? px : y.x, ly = upper ? py : y.y;
                const float bx = upper ? y.x : px, by = upper ? y.y : py;
                const float tr = __fmaf_rn(bx, w[s - 1].x, -__fmul_rn(by, w[s - 1].y));
                const float ti = __fmaf_rn(bx, w[s - 1].y, __fmul_rn(by, w[s - 1].x));
                y = upper ? make_float2(__fsub_rn(lx, tr), __fsub_rn(ly, ti))
                          : make_float2(__fadd_rn(lx, tr), __fadd_rn(ly, ti));
            }
            const long long s = s0 + tau0 + u;
            if (s < s1)
                __stcs(out + s * N + bin, y);
        }
    }
}

} // namespace ppfg

namespace ppfg {

// K6 at C = 1 (the FIR alone; the 1-point FFT is the identity): lanes take
// CONSECUTIVE output spectra instead of separate segments, so every load and
// store of a warp is one contiguous 256-byte run. Each warp walks its segment
// 32 spectra per step: it loads the next 32 input samples (coalesced) into a
// per-warp ring of 3 x 32 samples in shared memory (converted to double once
// on arrival), and lane l filters
// y[s0 + l] = sum_t h[t] x[s0 + l + t] from the ring (consecutive lanes read
// consecutive samples: conflict-free), in FP64 in ascending tap order from
// h0*x0 — bit-identical to ppf_fir_optimized (fir.hpp:85-110). T <= 33.
template <int T>
__global__ void __launch_bounds__(256) fir_c1_kernel(const float2* __restrict__ in,
                                                     float2* __restrict__ out, long long S_in,
                                                     long long S_out, const float* __restrict__ taps,
                                                     int seg, long long n_tasks) {
    static_assert(T >= 1 && T <= 33, "a window spans at most two 32-sample chunks");
    __shared__ double2 ring_s[8][96]; // converted once on arrival, read T times
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (task >= n_tasks)
        return;
    double2* ring = ring_s[wib];
    const long long s0 = task * seg;
    const long long s1 = min(s0 + seg, S_out);
    double h[T];
#pragma unroll
    for (int t = 0; t < T; ++t)
        h[t] = static_cast<double>(__ldg(taps + t));
    auto ld = [&](long long i) { return i < S_in ? __ldcs(in + i) : make_float2(0.f, 0.f); };
    auto cvt = [](float2 v) { return make_double2(static_cast<double>(v.x), static_cast<double>(v.y)); };
    // chunk q (samples s0 + 32q ..) lives in ring slot q % 3
    ring[lane] = cvt(ld(s0 + lane));
    ring[32 + lane] = cvt(ld(s0 + 32 + lane));
    float2 next = ld(s0 + 64 + lane);
    int q = 0;
    for (long long s = s0; s < s1; s += 32, ++q) {
        __syncwarp();
        double ar, ai;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int i = lane + t; // chunk q (i < 32) or q + 1
            const double2 x = ring[((q + (i >> 5)) % 3) * 32 + (i & 31)];
            if (t == 0) {
                ar = __dmul_rn(h[0], x.x);
                ai = __dmul_rn(h[0], x.y);
            } else {
                ar = __fma_rn(h[t], x.x, ar);
                ai = __fma_rn(h[t], x.y, ai);
            }
        }
        if (s + lane < s1)
            __stcs(out + s + lane, make_float2(__double2float_rn(ar), __double2float_rn(ai)));
        __syncwarp();
        ring[((q + 2) % 3) * 32 + lane] = cvt(next); // chunk q + 2 replaces chunk q - 1
        next = ld(s + 96 + lane);
    }
}

} // namespace ppfg
