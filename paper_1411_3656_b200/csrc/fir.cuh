// fir.cuh — K1: the polyphase FIR stage, bit-exact to ppf_fir_optimized.
//
// Reference contract (fir.hpp:85-110, 158-212): y[s][c] = sum_t h[t][c] x[s+t][c]
// over valid windows, each output component accumulated in double as
// acc = h0*x0 (a product), then acc = fma(h_t, x_t, acc) for t = 1..T-1 in
// ascending order, then rounded to float. Taps are the f32-quantised values.
// Products of two floats are exact in double, so DMUL/DFMA on the same operands
// in the same order reproduce every bit, including the sign of exact zeros.
//
// Mapping: one thread per (channel, time segment). Lanes take consecutive
// channels, so each warp load/store of a spectrum row is one coalesced 256 B
// transaction. The thread keeps the T-spectrum window of its channel in
// registers (as doubles: each input is converted once, not T times) and
// slides it down the segment; the (T-1)-spectrum warm-up per segment is the
// halo and mostly hits L2.
#pragma once

#include "common.cuh"

namespace ppfg {

template <int T>
__global__ void __launch_bounds__(256) fir_exact_kernel(const float2* __restrict__ in,
                                                        float2* __restrict__ out, unsigned C,
                                                        long long S_out,
                                                        const float* __restrict__ taps, int seg,
                                                        long long n_work, double init) {
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= n_work)
        return;
    const unsigned c = static_cast<unsigned>(g % C);
    const long long s0 = (g / C) * seg;
    const long long s1 = min(s0 + seg, S_out);
    double h[T];
#pragma unroll
    for (int t = 0; t < T; ++t)
        h[t] = static_cast<double>(__ldg(taps + static_cast<size_t>(t) * C + c));
    const float2* src = in + s0 * C + c;
    float2* dst = out + s0 * C + c;
    double xr[T], xi[T];
#pragma unroll
    for (int t = 0; t + 1 < T; ++t) {
        const float2 x = __ldcs(src + static_cast<long long>(t) * C);
        xr[t + 1] = x.x;
        xi[t + 1] = x.y;
    }
    src += static_cast<long long>(T - 1) * C;
#pragma unroll 2
    for (long long s = s0; s < s1; ++s) {
#pragma unroll
        for (int t = 0; t + 1 < T; ++t) {
            xr[t] = xr[t + 1];
            xi[t] = xi[t + 1];
        }
        const float2 x = __ldcs(src);
        src += C;
        xr[T - 1] = x.x;
        xi[T - 1] = x.y;
        // init = -0.0: fma(h, x, -0) == h*x bit for bit (fir.hpp:92-93);
        // init = +0.0: the fma-from-zero start of ppf_fir_reference (fir.hpp:141-142)
        double ar = __fma_rn(h[0], xr[0], init);
        double ai = __fma_rn(h[0], xi[0], init);
#pragma unroll
        for (int t = 1; t < T; ++t) {
            ar = __fma_rn(h[t], xr[t], ar);
            ai = __fma_rn(h[t], xi[t], ai);
        }
        st_cs(dst, make_float2(__double2float_rn(ar), __double2float_rn(ai)));
        dst += C;
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
