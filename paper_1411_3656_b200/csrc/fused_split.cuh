// fused_split.cuh — K3s: the fused FIR+FFT for channel/tap counts whose FIR
// state does not fit one SM's register file (C >= 2048, T >= 16, FP64 at
// C = 1024), on a thread-block cluster of Q = 2^LQ CTAs (one per SM).
//
// The split is a transpose through distributed shared memory:
//  - FIR role of CTA r filters channels k*N/R + r*256 + j (k < R, j < 256)
//    of EVERY output spectrum of the cluster's range: each thread holds only
//    R = N/(Q*256) channels' windows and taps; they are exactly the labels
//    the first log2 R FFT stages pair, so the thread runs those stages in
//    registers (as in fused.cuh); and the CTA's input is R contiguous runs of
//    256 channels per spectrum, fetched by TMA bulk copies (cp.async.bulk,
//    SASS UBLKCP) into a local ring.
//  - FFT role of CTA d transforms the full C-point rows of batches
//    b = d, d+Q, d+2Q, ... (B spectra each): the remaining L - log2 R stages
//    in register passes of <= 5 label bits (fft.cuh; the swizzle is
//    bank-conflict-free for these schedules), with no cross-CTA FFT stage.
//  - The FIR writes batch b's outputs straight into its owner's tile: the
//    owner's own channels with st.shared, the other CTAs' with st.async
//    over DSMEM, whose bytes complete on the owner's full[t] mbarrier.
//
// Synchronisation per owner tile t (two tiles per CTA):
//   local FIR block written  : named barrier FULL[t] (FIR arrives, FFT syncs)
//   remote FIR blocks landed : full[t] mbarrier; the owner's FFT leader arms
//                              it (arrive.expect_tx of the Q-1 remote blocks)
//                              before it announces the tile free
//   tile t of CTA d free     : empty[d][t] mbarrier in every CTA, one remote
//                              arrive from d's FFT leader after its last read
// A cluster barrier after mbarrier init and before exit keeps every CTA's
// shared memory alive while others may still address it.
#pragma once

#include <cuda.h>

#include "cluster.cuh"

namespace ppfg {

// one predicated store, no branch: st.shared into this CTA's tile, or
// st.async into the owner's tile with its bytes completing on the owner's
// full[t] mbarrier. No "memory" clobber: the ring loads of later rows may be
// scheduled above it (the tile is never read by this role; ordering against
// the barrier operations, all volatile asm, is kept).
PPFG_DEV void st_local_or_async_f2(bool local, uint32_t laddr, uint32_t raddr, float2 v,
                                   uint32_t rbar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.u32 p, %0, 0;\n\t"
        "@p st.shared.v2.f32 [%1], {%3, %4};\n\t"
        "@!p st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%2], {%3, %4}, [%5];\n\t}" ::"r"(
            static_cast<uint32_t>(local)),
        "r"(laddr), "r"(raddr), "f"(v.x), "f"(v.y), "r"(rbar));
}

// "this warp has read its ring slot": its reads completed when their values
// were consumed, so no release semantics are needed — a release arrive would
// first wait for this thread's outstanding DSMEM stores
PPFG_DEV void mbar_arrive_relaxed(uint64_t* bar) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 3-D TMA tensor copy global -> this CTA's shared memory (SASS UTMALDG),
// completing its bytes on a local mbarrier
PPFG_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// move this warpgroup's register budget from the launch allocation to REGS
template <int REGS, int LAUNCH>
PPFG_DEV void set_max_regs() {
    if constexpr (REGS > LAUNCH)
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS));
    else if constexpr (REGS < LAUNCH)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS));
}

template <int L_, int LQ_, int T_, bool EXACT_, int FIR_WG_ = 2, int W_ = 5,
          int FIR_REGS_ = 152, int FFT_REGS_ = 104, int PC_ = 0, bool TW4_ = false, bool HS_ = false,
          bool PAIR_ = false, bool TRIV_ = false>
struct SplitCfg {
    // TRIV (FAST, R <= 4): the FIR role's prestages use their trivial
    // twiddles as additions (fused.cuh FusedCfg::TRIV)
    static constexpr bool TRIV = TRIV_;
    // PAIR: the FIR role filters two consecutive spectra per step with their
    // accumulation chains interleaved (each output still sums its taps in
    // ascending order, so results are unchanged): with R <= 2 channels per
    // thread a single chain per output leaves the FMA pipe waiting on its
    // own latency
    static constexpr bool PAIR = PAIR_;
    // HS: the owner tile is handed over per FFT warpgroup (pass group pg owns
    // rows [pg*B/2, (pg+1)*B/2)): local FULL named barrier, remote full
    // mbarrier and the empty mbarriers all per (tile, pass group), so a pass
    // group starts as soon as its half of the batch has landed and the FIR
    // role refills a half as soon as its pass group has read it (fused.cuh HS)
    static constexpr bool HS = HS_;
    static constexpr int PG = HS_ ? 2 : 1;
    // twiddle table element: float2 (wr, wi), or pre-expanded float4 (fft.cuh tw_load)
    static constexpr bool TW4 = TW4_;
    using TwT = typename std::conditional<TW4_, float4, float2>::type;
    static constexpr int L = L_, LQ = LQ_, T = T_;
    static constexpr bool EXACT = EXACT_;
    static constexpr int FIR_REGS = FIR_REGS_, FFT_REGS = FFT_REGS_;
    static constexpr int Q = 1 << LQ;
    static constexpr int N = 1 << L;
    static constexpr int NFIR = 128 * FIR_WG_, NFFT = 256, NT = NFIR + NFFT;
    static constexpr int R = N / (Q * NFIR); // channels per FIR thread
    static constexpr int RLOG = R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3;
    static constexpr int LREM = L - RLOG;    // stages left to the FFT role
    static constexpr int W = W_;
    static constexpr int WMAX = FftSchedule<LREM, W>::width(0);
    static constexpr int B = (NFFT << WMAX) / N > 0 ? (NFFT << WMAX) / N : 1; // spectra per batch
    static constexpr int BU = ilcm(B, T) / B; // batches per unrolled FIR body (window renaming)
    static constexpr int BQ = ilcm(BU, Q);    // n_batches granule: whole bodies, equal fills per CTA
    static constexpr int RUN = NFIR;          // channels per contiguous input run
    // the TMA view of the input: R runs of RUN channels (box {RUN, R, RB} at
    // {rank*RUN, 0, row}); a run longer than the 256-element box limit (R = 1
    // with 4 FIR warpgroups) is fetched as TSPLIT sub-runs of 256 instead
    // (view of N/256 runs, box {256, TSPLIT, RB} at {0, rank*TSPLIT, row})
    static constexpr int TSPLIT = RUN > 256 ? RUN / 256 : 1;
    static constexpr int MAP_RUN = TSPLIT > 1 ? 256 : RUN;
    static constexpr int MAP_R = TSPLIT > 1 ? N / 256 : R;      // runs in the view
    static constexpr int MAP_BOX_R = TSPLIT > 1 ? TSPLIT : R;   // runs per copy
    static constexpr unsigned STRIDE = sw_row_stride(N);
    static constexpr size_t TILE_FLOATS2 = size_t(B) * STRIDE;
    static constexpr size_t TILE_BYTES = sizeof(float2) * TILE_FLOATS2;
    // input ring: one chunk = RB spectra x R runs x RUN channels, ONE TMA
    // tensor copy (3-D box {RUN, R, RB} of 8-byte elements)
    static constexpr size_t AVAIL = 232448 - 2 * TILE_BYTES - 512;
    // twiddles in shared memory when that still leaves >= 48 KB of ring
    static constexpr bool TW_SMEM = sizeof(TwT) * N + 48 * 1024 <= AVAIL;
    static constexpr size_t TW_BYTES = TW_SMEM ? sizeof(TwT) * N : 0;
    static constexpr size_t RING_MAX = (AVAIL - TW_BYTES) < 96 * 1024 ? (AVAIL - TW_BYTES) : 96 * 1024;
    static constexpr size_t ROW_BYTES = sizeof(float2) * R * RUN; // one spectrum's runs
    // rows per chunk: the whole batch if two such chunks fit, else halves...
    static constexpr int RB = RING_MAX / (ROW_BYTES * B) >= 2 ? B
                              : (B % 2 == 0 && RING_MAX / (ROW_BYTES * (B / 2)) >= 2) ? B / 2
                                                                                        : 1;
    static constexpr size_t CHUNK_FLOATS2 = size_t(RB) * R * RUN;
    static constexpr size_t CHUNK_BYTES = sizeof(float2) * CHUNK_FLOATS2;
    static constexpr int PC = PC_ > 0 ? PC_ : int(RING_MAX / CHUNK_BYTES) < 64 ? int(RING_MAX / CHUNK_BYTES) : 64;
    static constexpr size_t RING_BYTES = CHUNK_BYTES * PC;
    static constexpr int PROWS = B / PG;      // tile rows per pass group
    static constexpr int PNT = NFFT / PG;     // threads per pass group
    static constexpr size_t BARS = sizeof(uint64_t) * (2 * PC + 2 * PG + 2 * Q * PG);
    static constexpr size_t RING_OFF = (TW_BYTES + 127) & ~size_t(127);
    static constexpr size_t TILE_OFF = RING_OFF + RING_BYTES;
    static constexpr size_t BAR_OFF = (TILE_OFF + 2 * TILE_BYTES + 7) & ~size_t(7);
    // ring_full[PC], ring_empty[PC], full[2][PG], empty[Q][2][PG]
    static constexpr size_t SMEM = BAR_OFF + BARS;
    static constexpr uint32_t REMOTE_BYTES = uint32_t(sizeof(float2)) * (Q - 1) * PROWS * (N / Q); // per pass group
    // detection (POWER): as fused.cuh — last-pass units per row, per-bin
    // accumulators when the FFT role's thread count is a multiple of it
    static constexpr int UL = N >> FftSchedule<LREM, W>::width(FftSchedule<LREM, W>::NP - 1);
    static constexpr bool POWER_OK = PNT % UL == 0;
    static constexpr int POWER_ROWS = PG * (PNT / UL);
    static_assert(!HS || B % 2 == 0, "HS splits the tile's rows over the two FFT warpgroups");
    static_assert(!PAIR || (B % 2 == 0 && RB % 2 == 0 && PROWS % 2 == 0 && T >= 2),
                  "spectrum pairs within a chunk and a pass group");
    static_assert(Q >= 2 && Q <= 8, "portable cluster sizes");
    static_assert(!TRIV || (!EXACT && RLOG >= 1 && RLOG <= 2), "trivial prestages: FAST, R = 2 or 4");
    static_assert(R >= 1 && R <= 8 && R * Q * NFIR == N, "every FIR thread owns whole channels");
    static constexpr int LAUNCH_REGS = (65536 / NT) & ~7;
    static_assert(FIR_REGS * NFIR + FFT_REGS * NFFT <= LAUNCH_REGS * NT, "register split");
    static_assert(SMEM <= 232448, "shared memory per CTA");
    static_assert(PC >= 2, "input ring too shallow");
    static_assert(B % RB == 0, "whole chunks per batch");
    static_assert(MAP_RUN <= 256 && MAP_BOX_R <= 256 && RB <= 256, "TMA box dimensions");
    static_assert(TSPLIT == 1 || (R == 1 && RUN % 256 == 0), "sub-run TMA view: one channel per thread");
    static_assert(BU * B <= 64, "FIR unroll too large");
};

// POWER: the detection variant — `out` receives per-CTA partial power sums
// (POWER_ROWS rows of N doubles per CTA) instead of the bins.
template <class Cfg, bool POWER = false>
__global__ void __launch_bounds__(Cfg::NT, 1)
    fused_split_kernel(const __grid_constant__ CUtensorMap in_map, const float2* __restrict__ in,
                       float2* __restrict__ out, long long S_out,
                       long long rows_per_cluster, const float* __restrict__ taps,
                       const typename Cfg::TwT* __restrict__ tw_g) {
    constexpr int T = Cfg::T, N = Cfg::N, R = Cfg::R, RLOG = Cfg::RLOG, Q = Cfg::Q;
    constexpr int NFIR = Cfg::NFIR, NFFT = Cfg::NFFT, NT = Cfg::NT, B = Cfg::B, PC = Cfg::PC;
    constexpr int BU = Cfg::BU, RUN = Cfg::RUN;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    using TwT = typename Cfg::TwT;
    TwT* tw_s = reinterpret_cast<TwT*>(smem_raw);
    float2* ring = reinterpret_cast<float2*>(smem_raw + Cfg::RING_OFF);
    float2* tiles = reinterpret_cast<float2*>(smem_raw + Cfg::TILE_OFF);
    uint64_t* ring_full = reinterpret_cast<uint64_t*>(smem_raw + Cfg::BAR_OFF);
    uint64_t* ring_empty = ring_full + PC;
    constexpr int PG = Cfg::PG, PROWS = Cfg::PROWS, PNT = Cfg::PNT;
    uint64_t* full = ring_empty + PC; // full[t * PG + pg]
    uint64_t* empty = full + 2 * PG;  // empty[(d * 2 + t) * PG + pg]

    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const long long cid = blockIdx.x / Q;
    const long long o0 = cid * rows_per_cluster;
    const long long o1 = min(o0 + rows_per_cluster, S_out);
    const long long rows = max(o1 - o0, 0LL);
    // whole unrolled bodies and equal fills per CTA: trailing batches are
    // padding rows, computed (from stale ring slots) and never stored
    const long long n_batches = ((rows + B - 1) / B + Cfg::BQ - 1) / Cfg::BQ * Cfg::BQ;

    if constexpr (Cfg::TW_SMEM) {
        for (int i = tid; i < N - 1; i += NT)
            tw_s[i] = tw_g[i];
    }
    if (tid < PC) {
        mbar_init(ring_full + tid, 1);
        mbar_init(ring_empty + tid, NFIR / 32);
    } else if (tid < PC + 2 * PG) {
        mbar_init(full + (tid - PC), 1);
    } else if (tid < PC + 2 * PG + 2 * Q * PG) {
        mbar_init(empty + (tid - PC - 2 * PG), 1);
    }
    fence_mbar_init();
    __syncthreads();
    if (tid == NFIR) { // arm both tiles (every pass group's half) for their first fill
        for (int i = 0; i < 2 * PG; ++i)
            mbar_arrive_expect_tx(full + i, Cfg::REMOTE_BYTES);
    }
    cluster_sync_all(); // every CTA's barriers exist before anyone addresses them

    if (tid >= NFIR) {
        // ================================ FFT role ================================
        set_max_regs<Cfg::FFT_REGS, Cfg::LAUNCH_REGS>();
        const int ftid = tid - NFIR;
        const int pg = ftid / PNT;            // pass group (HS), else 0
        const int ptid = ftid - pg * PNT;
        const TwT* tw = Cfg::TW_SMEM ? tw_s : tw_g;
        const long long n_fills = n_batches / Q;
        // detection accumulators (as fused.cuh): FP64 in EXACT mode, FP32 in
        // FAST mode flushed into the CTA's FP64 partial row every kFlush fills
        using PA = typename std::conditional<Cfg::EXACT, double, float>::type;
        constexpr long long kFlush = 16;
        constexpr int EL = POWER ? N / Cfg::UL : 1;
        PA pacc[EL];
#pragma unroll
        for (int k = 0; k < EL; ++k)
            pacc[k] = 0;
        double* part = nullptr;
        if constexpr (POWER) {
            static_assert(Cfg::POWER_OK, "per-bin accumulators");
            constexpr int UL = Cfg::UL;
            const int r = pg * (PNT / UL) + ptid / UL;
            const unsigned u = static_cast<unsigned>(ptid % UL);
            part = reinterpret_cast<double*>(out) +
                   (static_cast<size_t>(blockIdx.x) * Cfg::POWER_ROWS + r) * N + u;
        }
        bool flushed = false;
        auto flush = [&]() {
#pragma unroll
            for (int k = 0; k < EL; ++k) {
                double* d = part + crev(static_cast<unsigned>(k), Cfg::L);
                *d = (flushed ? *d : 0.0) + static_cast<double>(pacc[k]);
                pacc[k] = 0;
            }
            flushed = true;
        };
        for (long long f = 0; f < n_fills; ++f) {
            const int t = static_cast<int>(f & 1);
            const long long b = f * Q + rank;
            float2* tile = tiles + t * Cfg::TILE_FLOATS2 + pg * PROWS * Cfg::STRIDE;
            if (ftid == 0) PPFG_TR(1, f, 0);
            named_sync(1 + t * PG + pg, NFIR + PNT);                          // own block written
            if (ftid == 0) PPFG_TR(1, f, 1);
            mbar_wait(full + t * PG + pg, static_cast<uint32_t>((f >> 1) & 1)); // remote blocks landed
            if (ftid == 0) PPFG_TR(1, f, 2);
            FftPasses<Cfg::L, Cfg::LREM, Cfg::W, false, Cfg::TW_SMEM, PNT, 0, true, POWER>::run(
                nullptr, out, tile, Cfg::STRIDE, PROWS,
                OffsetRows{FusedRows{o0, o1, rows, b * B, B}, pg * PROWS}, tw, ptid,
                SyncNamed{1 + 2 * PG + pg, PNT}, pacc);
            named_sync(1 + 2 * PG + pg, PNT); // every read of the pass group's rows has completed
            if (ftid == 0) PPFG_TR(1, f, 3);
            if (ptid == 0) {
                mbar_arrive_expect_tx(full + t * PG + pg, Cfg::REMOTE_BYTES); // arm the next fill
                const uint32_t e = smem_u32(empty + (rank * 2 + t) * PG + pg);
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    mbar_arrive_remote_relaxed(mapa(e, static_cast<uint32_t>(q)));
            }
            if constexpr (POWER && !Cfg::EXACT) {
                if ((f + 1) % kFlush == 0)
                    flush();
            }
        }
        if constexpr (POWER)
            flush();
        cluster_sync_all();
        return;
    }

    // ================================== FIR role ==================================
    set_max_regs<Cfg::FIR_REGS, Cfg::LAUNCH_REGS>();
    using Acc = typename std::conditional<Cfg::EXACT, double, float>::type;
    using Win = typename std::conditional<Cfg::EXACT, double2, float2>::type;
    // thread j owns channels c_k = k*N/R + rank*RUN + j: the R labels the
    // first RLOG stages pair, and R contiguous runs of RUN channels per CTA
    const int j = tid;
    const bool producer = (j == 0);
    const bool warp_leader = (tid & 31) == 0;
    const float2* gsrc = in + o0 * N + rank * RUN; // run 0 of input spectrum o0 + q

    // chunk c = input spectra T-1 + c*RB .. +RB (their R runs of this CTA);
    // rows past the input's end are zero-filled by TMA (they feed only
    // padding outputs)
    const long long n_chunks = (rows + Cfg::RB - 1) / Cfg::RB;
    auto issue = [&](long long c, int slot) {
        mbar_arrive_expect_tx(ring_full + slot, static_cast<uint32_t>(Cfg::CHUNK_BYTES));
        tma_load_3d(ring + slot * Cfg::CHUNK_FLOATS2, &in_map,
                    Cfg::TSPLIT > 1 ? 0 : static_cast<int>(rank * RUN),
                    Cfg::TSPLIT > 1 ? static_cast<int>(rank * Cfg::TSPLIT) : 0,
                    static_cast<int>(o0 + T - 1 + c * Cfg::RB), ring_full + slot);
    };
    if (producer) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&in_map)) : "memory");
        for (long long c = 0; c < n_chunks && c < PC; ++c)
            issue(c, static_cast<int>(c));
    }
    // ring cursors: consumer (chunk c) and refill, slot + parity
    // (rc = next chunk to issue; it reuses the slot of chunk rc - PC)
    int cslot = 0, rslot = 0;
    uint32_t cphase = 0, rphase = 0;
    long long rc = PC;

    Acc h[R][T];
    Win xw[R][T];
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
            h[k][t] = static_cast<Acc>(
                __ldg(taps + static_cast<size_t>(t) * N + k * (N / R) + rank * RUN + j));
            float2 x = make_float2(0.f, 0.f);
            if (t >= 1 && rows > 0)
                x = __ldg(gsrc + static_cast<long long>(t - 1) * N + k * (N / R) + j);
            xw[k][t].x = static_cast<Acc>(x.x);
            xw[k][t].y = static_cast<Acc>(x.y);
        }
    }
    float4 twr[R > 1 ? R - 1 : 1];
#pragma unroll
    for (int i = 0; i + 1 < R; ++i)
        twr[i] = tw_load<false>(tw_g + i);

    // tile slot offsets (float2 units) of this thread's channels
    unsigned slot_of[R];
#pragma unroll
    for (int k = 0; k < R; ++k)
        slot_of[k] = sw(static_cast<unsigned>(k * (N / R) + rank * RUN + j));
    const uint32_t tiles_u32 = smem_u32(tiles);
    const uint32_t full_u32 = smem_u32(full);

    for (long long b0 = 0; b0 < n_batches; b0 += BU) {
#pragma unroll
        for (int u = 0; u < BU; ++u) {
            const long long b = b0 + u;
            const long long f = b / Q;            // owner's fill index
            const int d = static_cast<int>(b - f * Q); // owner CTA
            const int t = static_cast<int>(f & 1);     // owner's tile
            if (tid == 0) PPFG_TR(0, b, 0);
            if (!Cfg::HS && f >= 2)
                mbar_wait(empty + d * 2 + t, static_cast<uint32_t>(((f >> 1) - 1) & 1));
            if (tid == 0) PPFG_TR(0, b, 1);
            const bool local = (static_cast<uint32_t>(d) == rank);
            const uint32_t tile_u32 = tiles_u32 + static_cast<uint32_t>(t * Cfg::TILE_BYTES);
            const uint32_t rtile = mapa(tile_u32, static_cast<uint32_t>(d));
            const uint32_t rbar0 = mapa(full_u32 + t * PG * 8u, static_cast<uint32_t>(d));
            constexpr int CPB = B / Cfg::RB;       // chunks per batch
            const long long c0 = b * CPB;         // this batch's chunks c0 .. c0+CPB-1
            if (producer) {
                // refill every slot released by the previous batches (all FIR
                // warps are done with chunks < c0 once they have arrived).
                // No proxy fence: the slot's last generic accesses are reads
                // ordered by the empty mbarrier (as in CUTLASS's TMA
                // pipelines), and a fence here would wait for this thread's
                // outstanding DSMEM stores.
                while (rc < n_chunks && rc < c0 + PC) {
                    mbar_wait(ring_empty + rslot, rphase);
                    issue(rc, rslot);
                    ++rc;
                    if (++rslot == PC) {
                        rslot = 0;
                        rphase ^= 1u;
                    }
                }
            }
            if (tid == 0) PPFG_TR(0, b, 4);
            // wait for the batch's chunks up front, so the rows below form
            // one straight-line block the scheduler can interleave
            int slot[CPB];
#pragma unroll
            for (int i = 0; i < CPB; ++i) {
                slot[i] = cslot;
                if (c0 + i < n_chunks)
                    mbar_wait(ring_full + cslot, cphase);
                if (++cslot == PC) {
                    cslot = 0;
                    cphase ^= 1u;
                }
            }
            const uint32_t ltile_u32 = tile_u32;
            if (tid == 0) PPFG_TR(0, b, 2);
            if constexpr (Cfg::PAIR) {
#pragma unroll
                for (int i = 0; i < B; i += 2) {
                    if constexpr (Cfg::HS) { // the owner's pass group i / PROWS has read tile t
                        if (i % PROWS == 0 && f >= 2)
                            mbar_wait(empty + (d * 2 + t) * PG + i / PROWS,
                                      static_cast<uint32_t>(((f >> 1) - 1) & 1));
                    }
                    const uint32_t rbar = rbar0 + 8u * static_cast<uint32_t>(i / PROWS);
                    const float2* c0p = ring + slot[i / Cfg::RB] * Cfg::CHUNK_FLOATS2 +
                                        (i % Cfg::RB) * (R * RUN) + j;
                    const float2* c1p = ring + slot[(i + 1) / Cfg::RB] * Cfg::CHUNK_FLOATS2 +
                                        ((i + 1) % Cfg::RB) * (R * RUN) + j;
                    float2 y0[R], y1[R];
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        // window convention: xw[k][t] = x[i + t - 1], t = 1..T-1; output i
                        // reads (xw[1..T-1], a), output i+1 (xw[2..T-1], a, b)
                        const float2 xa = c0p[k * RUN], xb = c1p[k * RUN];
                        Win a, bb;
                        a.x = static_cast<Acc>(xa.x);
                        a.y = static_cast<Acc>(xa.y);
                        bb.x = static_cast<Acc>(xb.x);
                        bb.y = static_cast<Acc>(xb.y);
                        auto v0 = [&](int tt) -> Win { return tt + 1 <= T - 1 ? xw[k][tt + 1] : a; };
                        auto v1 = [&](int tt) -> Win {
                            return tt + 2 <= T - 1 ? xw[k][tt + 2] : (tt + 2 == T ? a : bb);
                        };
                        if constexpr (Cfg::EXACT) {
                            double ar0 = __dmul_rn(h[k][0], v0(0).x), ai0 = __dmul_rn(h[k][0], v0(0).y);
                            double ar1 = __dmul_rn(h[k][0], v1(0).x), ai1 = __dmul_rn(h[k][0], v1(0).y);
#pragma unroll
                            for (int tt = 1; tt < T; ++tt) {
                                ar0 = __fma_rn(h[k][tt], v0(tt).x, ar0);
                                ai0 = __fma_rn(h[k][tt], v0(tt).y, ai0);
                                ar1 = __fma_rn(h[k][tt], v1(tt).x, ar1);
                                ai1 = __fma_rn(h[k][tt], v1(tt).y, ai1);
                            }
                            y0[k] = make_float2(__double2float_rn(ar0), __double2float_rn(ai0));
                            y1[k] = make_float2(__double2float_rn(ar1), __double2float_rn(ai1));
                        } else {
                            float2 acc0 = mul2s(h[k][0], v0(0)), acc1 = mul2s(h[k][0], v1(0));
#pragma unroll
                            for (int tt = 1; tt < T; ++tt) {
                                acc0 = fma2s(h[k][tt], v0(tt), acc0);
                                acc1 = fma2s(h[k][tt], v1(tt), acc1);
                            }
                            y0[k] = acc0;
                            y1[k] = acc1;
                        }
#pragma unroll
                        for (int tt = 1; tt + 2 < T; ++tt)
                            xw[k][tt] = xw[k][tt + 2];
                        if (T >= 3)
                            xw[k][T - 2] = a;
                        xw[k][T - 1] = bb;
                    }
                    if constexpr (Cfg::TRIV) {
                        fft_prestages_trivial_r<RLOG>(y0);
                        fft_prestages_trivial_r<RLOG>(y1);
                    } else {
                        fft_prestages<Cfg::L, RLOG>(y0, twr);
                        fft_prestages<Cfg::L, RLOG>(y1, twr);
                    }
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const uint32_t off0 = 8u * (i * Cfg::STRIDE + slot_of[k]);
                        const uint32_t off1 = off0 + 8u * Cfg::STRIDE;
                        st_local_or_async_f2(local, ltile_u32 + off0, rtile + off0, y0[k], rbar);
                        st_local_or_async_f2(local, ltile_u32 + off1, rtile + off1, y1[k], rbar);
                    }
                    if constexpr (Cfg::HS) { // own block of pass group i / PROWS written
                        if (local && (i + 2) % PROWS == 0)
                            named_arrive(1 + t * PG + i / PROWS, NFIR + PNT);
                    }
                }
            } else {
    #pragma unroll
                for (int i = 0; i < B; ++i) {
                    if constexpr (Cfg::HS) { // the owner's pass group i / PROWS has read tile t
                        if (i % PROWS == 0 && f >= 2)
                            mbar_wait(empty + (d * 2 + t) * PG + i / PROWS,
                                      static_cast<uint32_t>(((f >> 1) - 1) & 1));
                    }
                    const uint32_t rbar = rbar0 + 8u * static_cast<uint32_t>(i / PROWS);
                    const float2* chunk = ring + slot[i / Cfg::RB] * Cfg::CHUNK_FLOATS2 +
                                          (i % Cfg::RB) * (R * RUN) + j;
                    float2 y[R];
    #pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const float2 x = chunk[k * RUN];
    #pragma unroll
                        for (int tt = 0; tt + 1 < T; ++tt)
                            xw[k][tt] = xw[k][tt + 1];
                        xw[k][T - 1].x = static_cast<Acc>(x.x);
                        xw[k][T - 1].y = static_cast<Acc>(x.y);
                        if constexpr (Cfg::EXACT) {
                            double ar = __dmul_rn(h[k][0], xw[k][0].x);
                            double ai = __dmul_rn(h[k][0], xw[k][0].y);
    #pragma unroll
                            for (int tt = 1; tt < T; ++tt) {
                                ar = __fma_rn(h[k][tt], xw[k][tt].x, ar);
                                ai = __fma_rn(h[k][tt], xw[k][tt].y, ai);
                            }
                            y[k] = make_float2(__double2float_rn(ar), __double2float_rn(ai));
                        } else {
                            float2 acc = mul2s(h[k][0], xw[k][0]);
    #pragma unroll
                            for (int tt = 1; tt < T; ++tt)
                                acc = fma2s(h[k][tt], xw[k][tt], acc);
                            y[k] = acc;
                        }
                    }
                    if constexpr (Cfg::TRIV)
                        fft_prestages_trivial_r<RLOG>(y);
                    else
                        fft_prestages<Cfg::L, RLOG>(y, twr);
    #pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const uint32_t off = 8u * (i * Cfg::STRIDE + slot_of[k]);
                        st_local_or_async_f2(local, ltile_u32 + off, rtile + off, y[k], rbar);
                    }
                    if constexpr (Cfg::HS) { // own block of pass group i / PROWS written
                        if (local && (i + 1) % PROWS == 0)
                            named_arrive(1 + t * PG + i / PROWS, NFIR + PNT);
                    }
                }
            }
            if (tid == 0) PPFG_TR(0, b, 3);
            __syncwarp();
            if (warp_leader) { // this warp is done with the batch's chunks
#pragma unroll
                for (int i = 0; i < CPB; ++i)
                    if (c0 + i < n_chunks)
                        mbar_arrive_relaxed(ring_empty + slot[i]);
            }
            if (!Cfg::HS && local)
                named_arrive(1 + t, NFIR + NFFT); // own block of tile t written
        }
    }
    cluster_sync_all();
}

} // namespace ppfg
