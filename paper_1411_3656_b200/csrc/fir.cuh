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

#include <cuda.h>

#include <type_traits>

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

// K1t — the same warp tasks and op sequence as fir_chain_kernel, with the
// input staged by TMA instead of register prefetch: each warp owns a private
// ring of NS chunks (RB spectra x CPW channels, one 2-D tensor copy each,
// SASS UTMALDG) in shared memory, refilled by its lane 0 as soon as the
// warp's lane-0 tap chunk has read a chunk's last spectrum — no cross-warp
// coupling. Freeing the prefetch registers lets two 8-warp blocks share an
// SM (the register-prefetch kernel needs ~218 registers at TC = 16, one
// block), and the ring keeps >= 2 chunks of lookahead in flight.
template <int TC, int K, int LAG, int RB>
struct FirTma {
    static constexpr int CPW = 32 / K;
    // rows a warp needs at once: the newest row of every tap chunk plus the
    // window prefill, rounded to chunks, plus two chunks of lookahead (not
    // rounded up to a power of two: at TC = 16 that would cost the second
    // block per SM its shared memory)
    static constexpr int SPAN = TC - 1 + (K - 1) * (TC - LAG);
    static constexpr int NS = (SPAN + TC) / RB + 3;
    static constexpr size_t RING_FLOATS2 = size_t(NS) * RB * CPW;
    static constexpr int WARPS = 8;
    static constexpr size_t BAR_OFF = sizeof(float2) * RING_FLOATS2 * WARPS;
    static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) * NS * WARPS;
};

template <int TC, int K, int LAG, int RB, int MINB>
__global__ void __launch_bounds__(256, MINB) fir_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                         float2* __restrict__ out, unsigned C,
                                                         long long S_out,
                                                         const float* __restrict__ taps, int seg,
                                                         long long n_tasks, double init) {
    using F = FirTma<TC, K, LAG, RB>;
    constexpr int CPW = F::CPW, NS = F::NS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    float2* ring = reinterpret_cast<float2*>(smem_raw) + warp * F::RING_FLOATS2;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + F::BAR_OFF) + warp * NS;
    const long long task = static_cast<long long>(blockIdx.x) * F::WARPS + warp;
    if (task >= n_tasks)
        return; // warps are independent: no block-wide barrier below
    const int q = lane / CPW;
    const int cl = lane - q * CPW;
    const long long n_cb = (C + CPW - 1) / CPW;
    const long long sg = task / n_cb;
    const unsigned c0 = static_cast<unsigned>((task - sg * n_cb) * CPW);
    const unsigned c_raw = c0 + cl;
    const bool live = q < K && c_raw < C;
    const unsigned c = live ? c_raw : 0u;
    const int qq = q < K ? q : K - 1;
    const long long s0 = sg * seg;
    const long long s1 = min(s0 + seg, S_out);
    const int steps = static_cast<int>(s1 - s0) + LAG * (K - 1);
    // relative rows rr = 0 .. n_rows-1 (absolute s0 + rr; TMA zero-fills past the input)
    const int n_rows = steps + TC - 1 + (K - 1) * (TC - LAG);
    const int n_chunks = (n_rows + RB - 1) / RB;

    if (lane == 0) {
        for (int i = 0; i < NS; ++i)
            mbar_init(full + i, 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int k) { // lane 0 only
        const int slot = k % NS;
        mbar_arrive_expect_tx(full + slot, static_cast<uint32_t>(sizeof(float2) * RB * CPW));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(ring + slot * RB * CPW)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(static_cast<int>(c0)),
            "r"(static_cast<int>(s0 + static_cast<long long>(k) * RB)), "r"(smem_u32(full + slot))
            : "memory");
    };
    if (lane == 0)
        for (int k = 0; k < NS && k < n_chunks; ++k)
            issue(k);
    int waited = 0;   // chunks [0, waited) have landed
    int released = 0; // chunks [0, released) are consumed; issued = released + NS
    auto wait_upto = [&](int rr) {
        const int k1 = min(rr / RB, n_chunks - 1);
        for (; waited <= k1; ++waited)
            mbar_wait(full + waited % NS, static_cast<uint32_t>((waited / NS) & 1));
    };
    auto row = [&](int rr) { // this lane's channel of relative row rr
        return ring[((rr / RB) % NS) * RB * CPW + (rr % RB) * CPW + cl];
    };

    double h[TC];
#pragma unroll
    for (int t = 0; t < TC; ++t)
        h[t] = static_cast<double>(__ldg(taps + static_cast<size_t>(qq * TC + t) * C + c));

    const int base = qq * (TC - LAG); // lane q's rows: base + tau + [0, TC)
    wait_upto(base + TC - 2 + (K - 1 - qq) * (TC - LAG));
    double2 w[TC];
#pragma unroll
    for (int t = 0; t + 1 < TC; ++t) {
        const float2 x = row(base + t);
        w[t] = make_double2(x.x, x.y);
    }
    const unsigned src_lane_off = CPW;
    double2 carry[LAG];
#pragma unroll
    for (int i = 0; i < LAG; ++i)
        carry[i] = make_double2(0.0, 0.0);
    for (int tau0 = 0; tau0 < steps; tau0 += TC) {
        // chunks wholly below lane 0's first read of this block were read
        // (and converted) in earlier blocks: refill their slots
        const int done = (tau0 + TC - 1) / RB;
        __syncwarp();
        for (; released < done; ++released)
            if (lane == 0 && released + NS < n_chunks)
                issue(released + NS);
        wait_upto(tau0 + 2 * TC - 2 + (K - 1) * (TC - LAG));
#pragma unroll
        for (int u = 0; u < TC; ++u) {
            const int tau = tau0 + u;
            const float2 xn = row(base + tau + TC - 1);
            w[(u + TC - 1) % TC] = make_double2(xn.x, xn.y);
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
            if (live && qq == K - 1 && tau < steps && s >= s0 && s < s1)
                __stcs(out + s * C + c, make_float2(__double2float_rn(acc.x),
                                                    __double2float_rn(acc.y)));
        }
    }
}

// K1f — FIR in FP32 for PPFG_FAST's unfused path (T > 16, where no fused
// kernel exists): K lanes per channel each own TC consecutive taps and
// accumulate their partial sum with packed FFMA2 (re and im together); the K
// partials are added in a fixed tree order with shuffles. Not bit-exact by
// design (reassociated FP32 sum; max|err|/RMS ~1e-6, inside the FAST
// tolerance); ppfg_fir itself always runs the exact K1/K1t. Input staged by
// TMA in a per-warp ring as in K1t.
template <int TC, int K, int RB>
struct FirFast {
    static_assert(TC % 2 == 0 && (K & (K - 1)) == 0, "even tap chunks, power-of-two lanes");
    static constexpr int CPW = 32 / K;
    static constexpr int SPAN = TC - 1 + (K - 1) * TC;
    static constexpr int NS_MIN = (SPAN + TC) / RB + 3;
    // a power of two, so slot and parity are masks and shifts
    static constexpr int NS = NS_MIN <= 4 ? 4 : NS_MIN <= 8 ? 8 : NS_MIN <= 16 ? 16 : 32;
    static constexpr size_t RING_FLOATS2 = size_t(NS) * RB * CPW;
    static constexpr int WARPS = 8;
    static constexpr size_t BAR_OFF = sizeof(float2) * RING_FLOATS2 * WARPS;
    static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) * NS * WARPS;
};

template <int TC, int K, int RB>
__global__ void __launch_bounds__(256, 3) fir_fast_kernel(const __grid_constant__ CUtensorMap map,
                                                          float2* __restrict__ out, unsigned C,
                                                          long long S_out,
                                                          const float* __restrict__ taps, int seg,
                                                          long long n_tasks) {
    using F = FirFast<TC, K, RB>;
    constexpr int CPW = F::CPW, NS = F::NS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    float2* ring = reinterpret_cast<float2*>(smem_raw) + warp * F::RING_FLOATS2;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + F::BAR_OFF) + warp * NS;
    const long long task = static_cast<long long>(blockIdx.x) * F::WARPS + warp;
    if (task >= n_tasks)
        return;
    const int q = lane / CPW;
    const int cl = lane - q * CPW;
    const long long n_cb = (C + CPW - 1) / CPW;
    const long long sg = task / n_cb;
    const unsigned c0 = static_cast<unsigned>((task - sg * n_cb) * CPW);
    const unsigned c_raw = c0 + cl;
    const bool live = q < K && c_raw < C;
    const unsigned c = live ? c_raw : 0u;
    const int qq = q < K ? q : K - 1;
    const long long s0 = sg * seg;
    const long long s1 = min(s0 + seg, S_out);
    const int steps = static_cast<int>(s1 - s0);
    const int n_rows = steps + F::SPAN;
    const int n_chunks = (n_rows + RB - 1) / RB;

    if (lane == 0) {
        for (int i = 0; i < NS; ++i)
            mbar_init(full + i, 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int k) {
        const int slot = k % NS;
        mbar_arrive_expect_tx(full + slot, static_cast<uint32_t>(sizeof(float2) * RB * CPW));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(ring + slot * RB * CPW)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(static_cast<int>(c0)),
            "r"(static_cast<int>(s0 + static_cast<long long>(k) * RB)), "r"(smem_u32(full + slot))
            : "memory");
    };
    if (lane == 0)
        for (int k = 0; k < NS && k < n_chunks; ++k)
            issue(k);
    int waited = 0, released = 0;
    auto wait_upto = [&](int rr) {
        const int k1 = min(rr / RB, n_chunks - 1);
        for (; waited <= k1; ++waited)
            mbar_wait(full + waited % NS, static_cast<uint32_t>((waited / NS) & 1));
    };
    auto row = [&](int rr) { return ring[((rr / RB) % NS) * RB * CPW + (rr % RB) * CPW + cl]; };

    float h[TC];
#pragma unroll
    for (int t = 0; t < TC; ++t)
        h[t] = __ldg(taps + static_cast<size_t>(qq * TC + t) * C + c);
    const int base = qq * TC; // lane q's rows for output s0+tau: base + tau + [0, TC)
    wait_upto(F::SPAN - 1);
    float2 w[TC];
#pragma unroll
    for (int t = 0; t + 1 < TC; ++t)
        w[t] = row(base + t);
    for (int tau0 = 0; tau0 < steps; tau0 += TC) {
        const int done = (tau0 + TC - 1) / RB;
        __syncwarp();
        for (; released < done; ++released)
            if (lane == 0 && released + NS < n_chunks)
                issue(released + NS);
        wait_upto(tau0 + TC - 1 + F::SPAN);
#pragma unroll
        for (int u = 0; u < TC; ++u) {
            const int tau = tau0 + u;
            w[(u + TC - 1) % TC] = row(base + tau + TC - 1);
            // two interleaved partial sums (even / odd taps) halve the
            // dependent FFMA2 chain
            float2 acc = mul2s(h[0], w[u % TC]);
            float2 acc1 = mul2s(h[1], w[(u + 1) % TC]);
#pragma unroll
            for (int t = 2; t < TC; t += 2) {
                acc = fma2s(h[t], w[(u + t) % TC], acc);
                acc1 = fma2s(h[t + 1], w[(u + t + 1) % TC], acc1);
            }
            acc = add2(acc, acc1);
#pragma unroll
            for (int off = (K / 2) * CPW; off >= CPW; off >>= 1) {
                acc.x += __shfl_down_sync(0xffffffffu, acc.x, off);
                acc.y += __shfl_down_sync(0xffffffffu, acc.y, off);
            }
            const long long s = s0 + tau;
            if (live && q == 0 && tau < steps)
                __stcs(out + s * C + c, acc);
        }
    }
}

// Any T: the same op sequence, window re-read through L1/L2 per tap.
static __global__ void __launch_bounds__(256) fir_exact_generic_kernel(const float2* __restrict__ in,
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


// K1b — register-blocked FIR for long filters (T >= 16), exact (FP64, the
// reference's per-output op sequence) or FP32 (PPFG_FAST). A CTA of NW warps
// owns 32 consecutive channels (lane = channel) of one time segment and
// streams its input rows through a CTA-wide shared-memory ring of chunks of
// RB = NW*U rows (one 2-D TMA tensor copy each, SASS UTMALDG). Per step,
// warp w computes the U consecutive outputs [k*RB + w*U, +U) of its lane's
// channel: it reads each of the U+T-1 input rows it needs ONCE from shared
// memory and applies it to all U accumulators that use it (output u takes row
// j with tap j-u), taps held in registers. So an input row costs one LDS.64
// per U outputs' worth of taps — no register window rotation and no lane
// shuffles (K1's chain and K1f's tree) — and each output still accumulates
// its taps in ascending order: acc = fma(h_0, x_0, init) then fma(h_t, x_t,
// acc), i.e. bit-identical to ppf_fir_optimized (fir.hpp:85-110) in the
// exact mode. The FP32 mode runs the same chain in packed FFMA2 (re and im
// of one sample with the tap as a broadcast operand).
//
// FFA (FP32 only, PPFG_FAST fir+fft): the 2-parallel fast FIR algorithm.
// With he[k] = h[2k], ho[k] = h[2k+1] and, for output pair s = r0 + 2m,
//   A[m] = sum_k he[k] x[s+2k],  B[m] = sum_k ho[k] x[s+2k+1],
//   P[m] = sum_k (he[k]+ho[k]) (x[s+2k+1] + x[s+2k+2]),
// y[s] = A[m] + B[m] and y[s+1] = P[m] - (A[m+1] + B[m]): three T/2-tap
// filters per two outputs instead of two T-tap ones — 0.84-0.87x the FMA-pipe
// work at T = 32..64 counting the pre- and post-additions. Another rounding
// than the reference's ascending chain (inside the FAST fir+fft tolerance).
template <int T, int U, int NW, bool EXACT>
struct FirBlk {
    static constexpr int NT = NW * 32;
    static constexpr int RB = NW * U;                        // rows per chunk = per step
    static constexpr int NEED = 1 + (T - 1 + RB - 1) / RB;   // chunks one step reads
    static constexpr int NS_MIN = NEED + 2;                  // + two chunks of lookahead
    static constexpr int NS = NS_MIN <= 4 ? 4 : NS_MIN <= 8 ? 8 : 16;
    static constexpr int NR = NS * RB;                       // ring rows (power of two)
    static constexpr size_t CHUNK_BYTES = sizeof(float2) * RB * 32;
    static constexpr size_t BAR_OFF = sizeof(float2) * size_t(NR) * 32;
    static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) * NS;
    static_assert((RB & (RB - 1)) == 0 && RB <= 256, "power-of-two chunks within a TMA box");
};

template <int T, int U, int NW, bool EXACT, int MINB, bool FFA = false>
__global__ void __launch_bounds__(NW * 32, MINB) fir_block_kernel(const __grid_constant__ CUtensorMap map,
                                                                  float2* __restrict__ out, unsigned C,
                                                                  long long S_out,
                                                                  const float* __restrict__ taps,
                                                                  int seg, double init) {
    using F = FirBlk<T, U, NW, EXACT>;
    constexpr int RB = F::RB, NS = F::NS, NR = F::NR, NEED = F::NEED;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2* ring = reinterpret_cast<float2*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + F::BAR_OFF);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const long long n_cb = (C + 31) / 32;
    const long long sg = blockIdx.x / n_cb;
    const unsigned c0 = static_cast<unsigned>((blockIdx.x - sg * n_cb) * 32);
    const bool live = c0 + lane < C;
    const unsigned c = live ? c0 + lane : C - 1;
    const long long s0 = sg * seg;
    const int rows = static_cast<int>(min(s0 + seg, S_out) - s0);
    const int n_steps = (rows + RB - 1) / RB;
    // chunks holding rows [0, rows + T - 1) (TMA zero-fills past the input)
    const int n_chunks = (rows + T - 1 + RB - 1) / RB;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i)
            mbar_init(full + i, 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int k) { // thread 0 only
        const int slot = k & (NS - 1);
        mbar_arrive_expect_tx(full + slot, static_cast<uint32_t>(F::CHUNK_BYTES));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(ring + slot * RB * 32)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(static_cast<int>(c0)),
            "r"(static_cast<int>(s0 + static_cast<long long>(k) * RB)), "r"(smem_u32(full + slot))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < NS && k < n_chunks; ++k)
            issue(k);

    static_assert(!FFA || (!EXACT && T % 2 == 0 && U % 2 == 0), "fast FIR: FP32, even T and U");
    using acc_t = typename std::conditional<EXACT, double2, float2>::type;
    using tap_t = typename std::conditional<EXACT, double, float>::type;
    constexpr int TT = FFA ? 1 : T; // the direct form's taps
    constexpr int TF = FFA ? T / 2 : 1; // the fast form's sub-filter taps
    tap_t h[TT];
    float he[TF], ho[TF], hs[TF];
    if constexpr (FFA) {
#pragma unroll
        for (int k = 0; k < T / 2; ++k) {
            he[k] = __ldg(taps + static_cast<size_t>(2 * k) * C + c);
            ho[k] = __ldg(taps + static_cast<size_t>(2 * k + 1) * C + c);
            hs[k] = __fadd_rn(he[k], ho[k]);
        }
    } else {
#pragma unroll
        for (int t = 0; t < T; ++t)
            h[t] = static_cast<tap_t>(__ldg(taps + static_cast<size_t>(t) * C + c));
    }

    int waited = 0;
    for (int k = 0; k < n_steps; ++k) {
        if (k > 0) {
            // every warp is done with step k-1, the last reader of chunk k-1
            __syncthreads();
            if (threadIdx.x == 0 && k - 1 + NS < n_chunks)
                issue(k - 1 + NS);
        }
        const int need = min(k + NEED - 1, n_chunks - 1);
        for (; waited <= need; ++waited)
            mbar_wait(full + (waited & (NS - 1)), static_cast<uint32_t>((waited / NS) & 1));

        const int r0 = k * RB + warp * U;
        // byte offset of (row r0, this lane) in the ring; rows wrap modulo NR
        const uint32_t base = smem_u32(ring);
        const uint32_t off0 = static_cast<uint32_t>(r0) * 256u + static_cast<uint32_t>(lane) * 8u;
        if constexpr (FFA) {
            constexpr int M = U / 2;
            float2 A[M + 1], Bq[M], P[M];
#pragma unroll
            for (int m = 0; m <= M; ++m)
                A[m] = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = 0; m < M; ++m) {
                Bq[m] = make_float2(0.f, 0.f);
                P[m] = make_float2(0.f, 0.f);
            }
            float2 xo_prev = make_float2(0.f, 0.f);
            auto row = [&](int j) {
                const uint32_t off = (off0 + static_cast<uint32_t>(j) * 256u) & (uint32_t(NR) * 256u - 1u);
                float2 x;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y) : "r"(base + off));
                return x;
            };
#pragma unroll
            for (int n = 0; n <= M + T / 2 - 1; ++n) {
                const float2 xe = row(2 * n); // x[r0 + 2n]
                if (n >= 1) {                 // q[n-1] = x[2n-1] + x[2n] -> P[m], k = n-1-m
                    const float2 q = add2(xo_prev, xe);
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const int kk = n - 1 - m;
                        if (kk >= 0 && kk < T / 2)
                            P[m] = fma2s(hs[kk], q, P[m]);
                    }
                }
#pragma unroll
                for (int m = 0; m <= M; ++m) { // A[m], k = n-m
                    const int kk = n - m;
                    if (kk >= 0 && kk < T / 2)
                        A[m] = fma2s(he[kk], xe, A[m]);
                }
                if (2 * n + 1 <= U + T - 3) {
                    const float2 xo = row(2 * n + 1); // x[r0 + 2n + 1] -> B[m], k = n-m
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const int kk = n - m;
                        if (kk >= 0 && kk < T / 2)
                            Bq[m] = fma2s(ho[kk], xo, Bq[m]);
                    }
                    xo_prev = xo;
                }
            }
#pragma unroll
            for (int m = 0; m < M; ++m) {
                const float2 ye = add2(A[m], Bq[m]);
                const float2 yo = sub2(P[m], add2(A[m + 1], Bq[m]));
                if (live && r0 + 2 * m < rows)
                    __stcs(out + (s0 + r0 + 2 * m) * C + c, ye);
                if (live && r0 + 2 * m + 1 < rows)
                    __stcs(out + (s0 + r0 + 2 * m + 1) * C + c, yo);
            }
        } else {
        acc_t acc[U];
#pragma unroll
        for (int j = 0; j < U + T - 1; ++j) {
            const uint32_t off = (off0 + static_cast<uint32_t>(j) * 256u) & (uint32_t(NR) * 256u - 1u);
            float2 x;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y) : "r"(base + off));
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = j - u;
                if (t < 0 || t >= T)
                    continue;
                if constexpr (EXACT) {
                    const double xr = static_cast<double>(x.x), xi = static_cast<double>(x.y);
                    if (t == 0) {
                        acc[u].x = __fma_rn(h[0], xr, init);
                        acc[u].y = __fma_rn(h[0], xi, init);
                    } else {
                        acc[u].x = __fma_rn(h[t], xr, acc[u].x);
                        acc[u].y = __fma_rn(h[t], xi, acc[u].y);
                    }
                } else {
                    if (t == 0)
                        acc[u] = mul2s(h[0], x);
                    else
                        acc[u] = fma2s(h[t], x, acc[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (live && r0 + u < rows) {
                float2 y;
                if constexpr (EXACT)
                    y = make_float2(__double2float_rn(acc[u].x), __double2float_rn(acc[u].y));
                else
                    y = acc[u];
                __stcs(out + (s0 + r0 + u) * C + c, y);
            }
        }
        } // direct form
    }
}

} // namespace ppfg
