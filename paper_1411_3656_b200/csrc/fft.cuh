// fft.cuh — the reference's radix-2 DIT FFT (dft.hpp:72-148), bit-exact, as a
// register/shared-memory pass engine for sm_100a.
//
// Formulation. The reference bit-reverses a row, then runs stages
// len = 2, 4, ..., N; stage s (half h = 2^{s-1}) pairs positions p, p + h and
// uses twiddle tw[h-1+j], j = p mod h (dft.hpp:113-133). Track each element by
// its LABEL n = rev_L(p) instead (the channel index it started from): stage s
// pairs labels differing in bit b = L - s, and j = rev_{s-1}(n >> (b+1)). After
// the last stage label n holds bin rev_L(n). So a thread that holds the 2^W
// elements whose labels differ only in bits [LO, LO+W) can run those W stages
// in registers, with exactly the reference's butterflies and twiddles, and
// element-wise results are bit-identical to FftPlan::transform.
//
// A row is processed in passes of <= W label bits from the top bit down.
// Between passes elements go through shared memory at swizzled slot sw(label).
// Unit (thread task) mapping per pass:
//   first pass  : fixed label bits [0, LO) = u  -> lanes read consecutive
//                 channels of the input row (coalesced 8-byte loads);
//   middle pass : fixed bits = (low LO bits of u) | (rest of u above the pass);
//   final pass  : fixed bits [W, L) = rev(u), so element k is bin u + rev_L(k)
//                 and lanes store consecutive bins (coalesced).
#pragma once

#include "common.cuh"

namespace ppfg {

// Twiddles are stored either as float2 (wr, wi) — the reference's f32 table
// entry tw[h-1+j] (dft.hpp:93-96) — expanded to the packed butterfly's
// operand after the load (common.cuh tw_expand), or pre-expanded as float4
// (wr, wi, -wi, wr): half the shared-memory bytes vs two fewer instructions
// per twiddle, chosen per kernel by measurement.
template <bool TW_SMEM>
PPFG_DEV float4 tw_load(const float2* p) {
    if constexpr (TW_SMEM)
        return tw_expand(*p);
    else
        return tw_expand(__ldg(p));
}
// float2 twiddles in shared memory read with a volatile load: kept in program
// order, so the compiler does not hoist a whole pass's twiddles into registers
// (K2n's 5-bit passes would otherwise need ~200 registers)
struct TwV2 {
    float x, y;
};
template <bool TW_SMEM>
PPFG_DEV float4 tw_load(const TwV2* p) {
    static_assert(TW_SMEM, "shared-memory twiddles only");
    float2 w;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(w.x), "=f"(w.y) : "r"(smem_u32(p)));
    return tw_expand(w);
}
template <bool TW_SMEM>
PPFG_DEV float4 tw_load(const float4* p) {
    if constexpr (TW_SMEM)
        return *p;
    else
        return __ldg(p);
}

// Stages for label bits [LO, LO+W), high bit first. v[k] has label fixed|k<<LO.
template <int L, int LO, int W, bool TW_SMEM, class TW>
PPFG_DEV void fft_stages(float2 (&v)[1 << W], unsigned fixed, const TW* __restrict__ tw) {
#pragma unroll
    for (int bb = W - 1; bb >= 0; --bb) {
        const int b = LO + bb;
        const int s = L - b;
        const unsigned half = 1u << (s - 1);
        const unsigned jf = (s > 1) ? (__brev(fixed >> (b + 1)) >> (33 - s)) : 0u;
        const TW* twb = tw + (half - 1) + jf;
#pragma unroll
        for (int k = 0; k < (1 << W); ++k) {
            if (k & (1 << bb))
                continue;
            const unsigned jk = crev((static_cast<unsigned>(k) << LO) >> (b + 1), s - 1);
            const float4 w = tw_load<TW_SMEM>(twb + jk);
            bfly2(v[k], v[k | (1 << bb)], w);
        }
    }
}

// The first RLOG stages (label bits L-1 .. L-RLOG) on a thread's R values
// whose labels are j + k*N/R: their twiddle index j_f is 0, so every thread
// needs exactly tw[0 .. R-2], passed in registers (twr).
template <int L, int RLOG>
PPFG_DEV void fft_prestages(float2 (&v)[1 << RLOG], const float4 (&twr)[RLOG > 0 ? (1 << RLOG) - 1 : 1]) {
#pragma unroll
    for (int bb = RLOG - 1; bb >= 0; --bb) {
        const int b = L - RLOG + bb;
        const int s = L - b;
        const int half = 1 << (s - 1);
#pragma unroll
        for (int k = 0; k < (1 << RLOG); ++k) {
            if (k & (1 << bb))
                continue;
            const unsigned jk = crev((static_cast<unsigned>(k) << (L - RLOG)) >> (b + 1), s - 1);
            bfly2(v[k], v[k | (1 << bb)], twr[half - 1 + jk]);
        }
    }
}

// FAST mode only: the same first two stages for R = 4 values (labels j,
// j + N/4, j + N/2, j + 3N/4) with their exact twiddles 1 (stage 1), 1 and -i
// (stage 2) applied as additions: 6 packed adds + 4 scalar adds instead of 4
// butterflies (the reference multiplies by the f32-rounded table entries,
// e.g. (6.1e-17, -1) for -i: a 1e-16-relative difference).
PPFG_DEV void fft_prestages_trivial(float2 (&v)[4]) {
    // stage 1 (label bit L-1): pairs (0, 2), (1, 3), twiddle 1
    const float2 a0 = add2(v[0], v[2]), a2 = sub2(v[0], v[2]);
    const float2 a1 = add2(v[1], v[3]), a3 = sub2(v[1], v[3]);
    // stage 2 (label bit L-2): (0, 1) twiddle 1; (2, 3) twiddle -i: t = (hi.y, -hi.x)
    v[0] = add2(a0, a1);
    v[1] = sub2(a0, a1);
    v[2] = make_float2(__fadd_rn(a2.x, a3.y), __fsub_rn(a2.y, a3.x));
    v[3] = make_float2(__fsub_rn(a2.x, a3.y), __fadd_rn(a2.y, a3.x));
}

// FAST mode: the prestages with their trivial twiddles as additions for any
// R <= 4 (R = 2: one stage, twiddle 1; R = 4: fft_prestages_trivial)
template <int RLOG>
PPFG_DEV void fft_prestages_trivial_r(float2 (&v)[1 << RLOG]) {
    if constexpr (RLOG == 1) {
        const float2 a = add2(v[0], v[1]), b = sub2(v[0], v[1]);
        v[0] = a;
        v[1] = b;
    } else if constexpr (RLOG == 2) {
        fft_prestages_trivial(v);
    }
}

// ---- pass schedule: NP passes of near-equal width, widest first ------------------
template <int L, int W>
struct FftSchedule {
    static constexpr int NP = L == 0 ? 1 : (L + W - 1) / W;
    __host__ __device__ static constexpr int width(int i) { return L / NP + (i < L % NP ? 1 : 0); }
    __host__ __device__ static constexpr int done(int i) {
        return i * (L / NP) + (i < L % NP ? i : L % NP);
    }
    __host__ __device__ static constexpr int lo(int i) { return L - done(i + 1); }
};

// One pass of the row engine over a tile of rows.
//   FIRST_GLOBAL: this (top) pass reads natural-order input rows from global.
//   FINAL       : this (bit-0) pass writes natural-order bins to global.
// map(r) gives the global row of tile row r, or -1 for a padding row.
// gin/gout may alias (in-place channelize): every row is fully read before it is
// written, with a barrier in between for multi-pass transforms.
// POWER (with FINAL): instead of storing the bins, add each bin's power
// p = (double)re*re + (double)im*im (cli.hpp:307-317) to the thread's
// accumulators pacc[k] — the caller guarantees one unit per thread, so
// pacc[k] always belongs to the same tile row and bin.
template <int L, int LO, int W, bool FIRST_GLOBAL, bool FINAL, bool TW_SMEM, int NT, bool POWER = false,
          class RowMap, class TW, class PA = double>
PPFG_DEV void fft_tile_pass(const float2* gin, float2* gout,
                            float2* __restrict__ tile, unsigned row_stride, int rows,
                            const RowMap& map, const TW* __restrict__ tw, int tid,
                            PA* pacc = nullptr) {
    constexpr int N = 1 << L;
    constexpr int E = 1 << W;
    constexpr int HI = LO + W - 1;
    constexpr int U = N >> W;
    static_assert(!FIRST_GLOBAL || HI == L - 1, "a global-source pass must be the top pass");
    static_assert(!FINAL || LO == 0, "the final pass ends at label bit 0");
    const int units = rows * U;
    for (int unit = tid; unit < units; unit += NT) {
        const int r = unit / U;
        const unsigned u = static_cast<unsigned>(unit % U);
        // a pass ending at label bit 0 maps lanes to the TOP label bits (bit-
        // reversed unit index): its outputs are then consecutive bins and its
        // twiddle reads consecutive table entries, whether it stores to global
        // (FINAL) or back to the tile for further (cross-CTA) stages.
        unsigned fixed;
        if constexpr (LO == 0)
            fixed = (L - W > 0) ? (crev_rt(u, L - W) << W) : 0u;
        else if constexpr (FIRST_GLOBAL)
            fixed = u;
        else
            fixed = (u & ((1u << LO) - 1u)) | ((u >> LO) << (HI + 1));
        float2 v[E];
        if constexpr (FIRST_GLOBAL) {
            const long long grow = map(r);
            const float2* src = gin + grow * N + fixed;
#pragma unroll
            for (int k = 0; k < E; ++k) // L2-only loads: the rows may have been written by other SMs
                v[k] = grow >= 0 ? __ldcg(src + (static_cast<unsigned>(k) << LO)) : make_float2(0.f, 0.f);
        } else {
            const float2* src = tile + r * row_stride + sw(fixed);
#pragma unroll
            for (int k = 0; k < E; ++k)
                v[k] = src[sw(static_cast<unsigned>(k) << LO)];
        }
        fft_stages<L, LO, W, TW_SMEM>(v, fixed, tw);
        if constexpr (FINAL && POWER) {
            if (map(r) >= 0) {
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    if constexpr (sizeof(PA) == 8)
                        pacc[k] += static_cast<double>(v[k].x) * v[k].x +
                                   static_cast<double>(v[k].y) * v[k].y;
                    else // FAST detection: FP32 partial sums, flushed to FP64 by the caller
                        pacc[k] = __fmaf_rn(v[k].x, v[k].x, __fmaf_rn(v[k].y, v[k].y, pacc[k]));
                }
            }
        } else if constexpr (FINAL) {
            const long long grow = map(r);
            if (grow >= 0) {
                float2* dst = gout + grow * N + u;
#pragma unroll
                for (int k = 0; k < E; ++k)
                    st_cs(dst + crev(static_cast<unsigned>(k), L), v[k]);
            }
        } else {
            float2* dst = tile + r * row_stride + sw(fixed);
#pragma unroll
            for (int k = 0; k < E; ++k)
                dst[sw(static_cast<unsigned>(k) << LO)] = v[k];
        }
    }
}

// The passes covering label bits [0, LREM) of an N = 2^L transform (the top
// L - LREM bits were already done, e.g. in the fused kernel's FIR threads).
// `tid` is the thread's index among the NT threads running the passes and
// `sync` the barrier between passes (__syncthreads, or a named barrier when
// only the FFT warps of a warp-specialised CTA take part).
// STORE_LAST = false keeps the last pass's results in the tile (swizzled, by
// label) instead of storing bins to global — used when more stages follow
// (the cluster kernel's cross-CTA stages).
// POWER: the last pass accumulates bin powers into pacc (see fft_tile_pass).
// LAST_GLOBAL: the last pass reads its twiddles from global memory (tw_last,
// the full table; its lanes read consecutive entries) while the earlier
// passes read `tw` — so a kernel needs only the first 2^(L - w_last) - 1
// entries in shared memory (K2n at C = 4096, 8192)
template <int L, int LREM, int W, bool FIRST_GLOBAL, bool TW_SMEM, int NT, int I = 0,
          bool STORE_LAST = true, bool POWER = false, bool LAST_GLOBAL = false>
struct FftPasses {
    using S = FftSchedule<LREM, W>;
    static constexpr int WI = S::width(I);
    static constexpr int LO = S::lo(I);
    static constexpr bool LAST = (I == S::NP - 1);
    static constexpr int E_LAST = 1 << S::width(S::NP - 1); // values per unit in the last pass
    template <class RowMap, class Sync, class TW, class PA = double>
    PPFG_DEV static void run(const float2* gin, float2* gout, float2* tile, unsigned row_stride,
                             int rows, const RowMap& map, const TW* tw, int tid,
                             const Sync& sync, PA* pacc = nullptr,
                             const float2* __restrict__ tw_last = nullptr) {
        if constexpr (LAST && LAST_GLOBAL)
            fft_tile_pass<L, LO, WI, FIRST_GLOBAL && I == 0, STORE_LAST, false, NT, POWER>(
                gin, gout, tile, row_stride, rows, map, tw_last, tid, pacc);
        else
            fft_tile_pass<L, LO, WI, FIRST_GLOBAL && I == 0, LAST && STORE_LAST, TW_SMEM, NT,
                          LAST && POWER>(gin, gout, tile, row_stride, rows, map, tw, tid, pacc);
        if constexpr (!LAST) {
            sync();
            FftPasses<L, LREM, W, FIRST_GLOBAL, TW_SMEM, NT, I + 1, STORE_LAST, POWER, LAST_GLOBAL>::run(
                gin, gout, tile, row_stride, rows, map, tw, tid, sync, pacc, tw_last);
        }
    }
};

struct SyncCta {
    PPFG_DEV void operator()() const { __syncthreads(); }
};

struct LinearRows {
    long long row0, n_rows;
    PPFG_DEV long long operator()(int r) const {
        return row0 + r < n_rows ? row0 + r : -1;
    }
};

// K2: channelize_block for power-of-two C = 2^L (L >= 1), rows independent.
// Persistent grid; each CTA transforms RB = max(1, NT*2^W/N) rows per tile.
template <int L, int W, bool TW_SMEM, int NT>
__global__ void __launch_bounds__(NT) fft_rows_kernel(const float2* in, float2* out,
                                                      long long n_rows,
                                                      const float2* __restrict__ tw_g) {
    constexpr int N = 1 << L;
    constexpr int RB = (NT << W) / N > 0 ? (NT << W) / N : 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2* tw_s = reinterpret_cast<float2*>(smem_raw);
    float2* tile = reinterpret_cast<float2*>(smem_raw + (TW_SMEM ? sizeof(float2) * N : 0));
    if constexpr (TW_SMEM) {
        for (int i = threadIdx.x; i < N - 1; i += NT)
            tw_s[i] = tw_g[i];
        __syncthreads();
    }
    const float2* tw = TW_SMEM ? tw_s : tw_g;
    constexpr unsigned stride = sw_row_stride(N);
    for (long long row0 = static_cast<long long>(blockIdx.x) * RB; row0 < n_rows;
         row0 += static_cast<long long>(gridDim.x) * RB) {
        FftPasses<L, L, W, true, TW_SMEM, NT>::run(in, out, tile, stride, RB,
                                                   LinearRows{row0, n_rows}, tw,
                                                   static_cast<int>(threadIdx.x), SyncCta{});
        __syncthreads();
    }
}

// K2n: channelize_block for 64 <= C <= 8192 as a NON-persistent grid of small
// CTAs, one tile of NR rows each (NR * C * 8 B = 16-64 KB), several CTAs per
// SM, dispatched in row order. Each CTA loads its rows with one TMA bulk copy
// per row into a swizzled-row slot, runs the first pass from the natural-order
// rows (one unit per thread: NT = NR * U0), writes it back in place at
// swizzled slots, then the remaining passes (FftPasses) and stores the bins.
// Twiddles: each CTA copies the table into shared memory while its rows land
// (read straight from global the compiler hoists a pass's twiddle loads and
// spills). Same
// butterflies as K2 / K3: bit-exact. The grid sweeps HBM as one narrow
// front, the access pattern that streamed fastest of everything measured here
// (profiles/round2/probes: a non-persistent block copy 6.78 TB/s vs 6.0-6.4
// persistent).
template <int L, int W, int NT, int UPT = 1, bool TWL = false>
struct FftTiles {
    using S = FftSchedule<L, W>;
    static constexpr int N = 1 << L;
    static constexpr int W0 = S::width(0), LO0 = S::lo(0);
    static constexpr int U0 = N >> W0;               // first-pass units per row
    static constexpr int NR = UPT * NT / U0;         // rows per CTA: UPT units per thread
    static constexpr unsigned STRIDE = sw_row_stride(N);
    // TWL: only the entries of the passes before the last in shared memory
    static constexpr int TW_N = TWL ? (1 << (L - S::width(S::NP - 1))) - 1 : N - 1;
    static constexpr size_t TW_BYTES = (sizeof(float2) * (TW_N + 1) + 127) & ~size_t(127);
    static constexpr size_t SMEM = TW_BYTES + sizeof(float2) * size_t(NR) * STRIDE;
    static_assert((UPT * NT) % U0 == 0 && NR >= 1, "whole rows of first-pass units");
    static_assert(S::NP >= 2, "pass 1 hands over to FftPasses<.., I = 1>");
};

template <int L, int W, int NT, int MINB = 1, int UPT = 1, bool VOLTW = false, bool TWL = false>
__global__ void __launch_bounds__(NT, MINB) fft_tiles_kernel(const float2* __restrict__ in,
                                                       float2* __restrict__ out, long long n_rows,
                                                       const float2* __restrict__ tw_g) {
    using F = FftTiles<L, W, NT, UPT, TWL>;
    using TWT = typename std::conditional<VOLTW, TwV2, float2>::type;
    constexpr int N = F::N, NR = F::NR, U0 = F::U0, W0 = F::W0, LO0 = F::LO0, E0 = 1 << W0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full;
    float2* tw = reinterpret_cast<float2*>(smem_raw);
    float2* slots = reinterpret_cast<float2*>(smem_raw + F::TW_BYTES);
    const int tid = threadIdx.x;
    const long long row0 = static_cast<long long>(blockIdx.x) * NR;
    const int rows = static_cast<int>(min(static_cast<long long>(NR), n_rows - row0));
    if (tid == 0) {
        mbar_init(&full, 1);
        fence_mbar_init();
    }
    __syncthreads();
    constexpr uint32_t ROW_BYTES = static_cast<uint32_t>(sizeof(float2) * N);
    if (tid == 0) {
        mbar_arrive_expect_tx(&full, ROW_BYTES * static_cast<uint32_t>(rows));
        for (int r = 0; r < rows; ++r)
            bulk_g2s(slots + r * F::STRIDE, in + (row0 + r) * N, ROW_BYTES, &full);
    }
    for (int i = tid; i < F::TW_N; i += NT)
        tw[i] = __ldg(tw_g + i);
    __syncthreads();
    mbar_wait(&full, 0);
    // pass 1 from the natural-order rows, written back in place (swizzled)
    float2 v[UPT][E0];
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
        const int u = tid + q * NT;
        const int r = u / U0;
        const unsigned fixed = static_cast<unsigned>(u % U0);
        if (r < rows) {
            const float2* slot = slots + r * F::STRIDE;
#pragma unroll
            for (int k = 0; k < E0; ++k)
                v[q][k] = slot[fixed + (static_cast<unsigned>(k) << LO0)];
            fft_stages<L, LO0, W0, true>(v[q], fixed, reinterpret_cast<const TWT*>(tw));
        }
    }
    __syncthreads(); // every natural-order read of the tile is done
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
        const int u = tid + q * NT;
        const int r = u / U0;
        const unsigned fixed = static_cast<unsigned>(u % U0);
        if (r < rows) {
            float2* dst = slots + r * F::STRIDE + sw(fixed);
#pragma unroll
            for (int k = 0; k < E0; ++k)
                dst[sw(static_cast<unsigned>(k) << LO0)] = v[q][k];
        }
    }
    __syncthreads();
    FftPasses<L, L, W, false, true, NT, 1, true, false, TWL>::run(
        nullptr, out, slots, F::STRIDE, rows, LinearRows{row0, n_rows},
        reinterpret_cast<const TWT*>(tw), tid, SyncCta{}, static_cast<double*>(nullptr), tw_g);
}

template <int L, int W, bool TW_SMEM, int NT>
constexpr size_t fft_rows_smem_bytes() {
    constexpr int N = 1 << L;
    constexpr int RB = (NT << W) / N > 0 ? (NT << W) / N : 1;
    constexpr bool multipass = FftSchedule<L, W>::NP > 1;
    return (TW_SMEM ? sizeof(float2) * N : 0) +
           sizeof(float2) * (multipass ? static_cast<size_t>(RB) * sw_row_stride(N) : 0);
}

} // namespace ppfg
