// dft.cuh — K4: dft_naive (dft.hpp:39-66) for non-power-of-two C, bit-exact,
// and K5: the counter-based synthetic input generator.
#pragma once

#include "common.cuh"

namespace ppfg {

// X[k] = sum_m x[m] * roots[(k*m) mod n] accumulated in double, one thread per
// (row, k). The reference's expression (dft.hpp:60-61) is contracted by GCC
// into acc += fma(xr, wr, -(xi*wi)) / acc += fma(xr, wi, xi*wr) when built the
// way proj/CMakeLists.txt builds it (pinned in tests/test_oracle.py); the same
// operations are written out here with _rn intrinsics.
static __global__ void __launch_bounds__(256) dft_naive_kernel(const float2* __restrict__ in,
                                                        float2* __restrict__ out, unsigned n,
                                                        long long n_rows,
                                                        const double2* __restrict__ roots) {
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= n_rows * n)
        return;
    const long long row = g / n;
    const unsigned k = static_cast<unsigned>(g % n);
    const float2* x = in + row * n;
    double ar = 0.0, ai = 0.0;
    unsigned idx = 0;
    for (unsigned m = 0; m < n; ++m) {
        const float2 v = __ldg(x + m);
        const double2 w = __ldg(roots + idx);
        const double xr = v.x, xi = v.y;
        ar = __dadd_rn(ar, __fma_rn(xr, w.x, -__dmul_rn(xi, w.y)));
        ai = __dadd_rn(ai, __fma_rn(xr, w.y, __dmul_rn(xi, w.x)));
        idx += k;
        if (idx >= n)
            idx -= n;
    }
    out[g] = make_float2(__double2float_rn(ar), __double2float_rn(ai));
}

// ---- synthetic tone + noise ---------------------------------------------------
// x[n] = tone[(f10 * n) mod (10 C)] + (g_re + i g_im): tone is a host-built f32
// table of e^{2 pi i k / (10 C)} (f = f10 / 10 = C/8 + 0.3 bins), g is an
// Irwin-Hall(4 x 16 bit) approximation of N(0,1) from splitmix64 keyed by the
// sample counter. Integer + IEEE-rounded float ops only => identical bytes on
// host (ppfg.cu, synth_host) and device.
PPFG_HD uint64_t splitmix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

PPFG_HD int irwin_hall4(uint64_t z) {
    return static_cast<int>((z & 0xffff) + ((z >> 16) & 0xffff) + ((z >> 32) & 0xffff) +
                            (z >> 48)) -
           131070;
}

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr float kNoiseScale = 2.64293e-05f; // 1 / sqrt(4 * (65536^2 - 1) / 12)

static __global__ void __launch_bounds__(256) synth_kernel(float2* __restrict__ out, uint64_t seed,
                                                    uint64_t first, uint64_t count, uint64_t f10,
                                                    uint64_t M, const float2* __restrict__ tone) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    const uint64_t n = first + i;
    const float2 t = __ldg(tone + (f10 * n) % M);
    const uint64_t a = splitmix64(seed + (2 * n + 1) * kGolden);
    const uint64_t b = splitmix64(seed + (2 * n + 2) * kGolden);
    const float gr = __fmul_rn(static_cast<float>(irwin_hall4(a)), kNoiseScale);
    const float gi = __fmul_rn(static_cast<float>(irwin_hall4(b)), kNoiseScale);
    out[i] = make_float2(__fadd_rn(t.x, gr), __fadd_rn(t.y, gi));
}

} // namespace ppfg
