// fused.cuh — K3: polyphase FIR + C-point FFT in one persistent,
// warp-specialised kernel (channelize_block(ppf_fir_optimized(x)),
// pipeline.hpp:125-127) with no HBM round trip for the filtered block.
//
// One CTA per SM owns a contiguous range of output spectra, split into G
// groups (G > 1 only for small C, so the FIR role always has 256 threads).
// Two roles run concurrently, handing tiles over through shared memory:
//
//  FIR role (warpgroups 0-1, setmaxnreg.inc): thread j of group g owns the
//    R = 2^RLOG channels j + k*N/R. Input spectra arrive in a P-slot TMA ring
//    (cp.async.bulk 1-D copies, SASS UBLKCP, one mbarrier per slot). Each
//    thread keeps its channels' T-spectrum windows and taps in registers,
//    slides them down the time axis (every input spectrum read once), and per
//    output spectrum runs the first RLOG radix-2 stages on its R values in
//    registers (they pair exactly those channels), then stores them to the
//    FFT tile at swizzled slots. Lane 0 of each group is the TMA producer:
//    once all FIR warps of the group have released ring slot q-D (per-slot
//    "empty" mbarrier), it refills that slot with spectrum q-D+P, so HBM
//    reads never wait for a batch boundary.
//
//  FFT role (warpgroups 2-3, setmaxnreg.dec): the remaining L-RLOG stages of
//    each tile in register passes of <= W = 4 bits through shared memory
//    (named barrier between passes, FFT warps only); the final pass stores
//    natural-order bins straight to HBM with coalesced 8-byte stores.
//
//  Handoff: two tiles; named barriers FULL[t] (FIR arrives, FFT syncs) and
//  EMPTY[t] (FFT arrives, FIR syncs), so the FIR of tile b+1 overlaps the FFT
//  of tile b.
//
// EXACT = true accumulates the FIR in FP64 in the reference order (bit-exact
// to ppf_fir_optimized); false accumulates in FP32, re and im together in one
// FFMA2 per tap. The FFT is always the reference's exact radix-2 arithmetic
// (packed FFMA2/FMUL2/FADD2, bit-identical, common.cuh bfly2).
#pragma once

#include <type_traits>

#include "fft.cuh"

namespace ppfg {

constexpr int ilcm(int a, int b) {
    int x = a, y = b;
    while (y) {
        const int t = x % y;
        x = y;
        y = t;
    }
    return a / x * b;
}

template <int L_, int T_, int RLOG_, bool EXACT_, int FIR_REGS_ = 160, int FFT_REGS_ = 96,
          int PC_ = 4, int FFT_WG_ = 2, int NTILE_ = 2, bool TW4_ = false, int L2A_ = 0,
          bool HS_ = false, bool TRIV_ = false, bool PAIR_ = false>
struct FusedCfg {
    // PAIR: two consecutive spectra per FIR step with interleaved accumulation
    // chains (same per-output operation order; fused_split.cuh SplitCfg::PAIR)
    static constexpr bool PAIR = PAIR_;
    // HS: hand tiles over per FFT pass group instead of whole: a FIR thread
    // arrives on FULL[t][pg] as soon as it has written its rows of pass group
    // pg and waits on EMPTY[t][pg] just before writing them, so each FFT
    // warpgroup starts on its rows while the FIR role is still filling the
    // rest (needs an evenly split tile; with several FIR groups a pass
    // group's barrier counts the groups that write its rows)
    static constexpr bool HS = HS_;
    // TRIV (FAST only): the FIR role's first two radix-2 stages use their
    // trivial twiddles (1, 1, -i) as additions instead of the reference's
    // multiplications by the rounded table values (6e-17 apart) — half the
    // FMA-pipe work of the prestages; EXACT keeps the reference arithmetic
    static constexpr bool TRIV = TRIV_;
    // L2A > 0: the producer also prefetches (cp.async.bulk.prefetch.L2) the
    // chunk L2A past the one it copies into the ring, so that chunk's bulk
    // copy later starts from L2 — lookahead without shared memory
    static constexpr int L2A = L2A_;
    // twiddle table element: float2 (wr, wi), or pre-expanded float4 (fft.cuh tw_load)
    static constexpr bool TW4 = TW4_;
    using TwT = typename std::conditional<TW4_, float4, float2>::type;
    static constexpr int NTILE = NTILE_; // FFT tiles in flight between the roles
    static constexpr int L = L_, T = T_, RLOG = RLOG_;
    static constexpr bool EXACT = EXACT_;
    static constexpr int FIR_REGS = FIR_REGS_, FFT_REGS = FFT_REGS_;
    static constexpr int N = 1 << L;
    static constexpr int R = 1 << RLOG;
    static constexpr int NTG = N / R;       // FIR threads per group
    static constexpr int NFIR = 256;        // FIR role: warpgroups 0-1
    static constexpr int NFFT = 128 * FFT_WG_; // FFT role: warpgroups 2 ..
    static constexpr int NT = NFIR + NFFT;
    static constexpr int G = NFIR / NTG;    // groups per CTA
    static constexpr int FW = NTG / 32;     // FIR warps per group
    static constexpr int W = 4;             // FFT pass width: 16 values per unit
    // spectra per group per batch (= per ring chunk and per tile): one FFT
    // unit per FFT thread per pass
    static constexpr int B = (NFFT << W) / (N * G) > 0 ? (NFFT << W) / (N * G) : 1;
    static constexpr int PC = PC_;          // ring chunks (of B input spectra) per group
    static constexpr int FFT_WG = FFT_WG_;
    // batches per unrolled FIR loop body, so the window rotation is pure renaming
    static constexpr int BU = ilcm(B, T) / B;
    static constexpr unsigned STRIDE = sw_row_stride(N);
    static constexpr size_t CHUNK_BYTES = sizeof(float2) * size_t(B) * N;
    // shared-memory layout (bytes)
    static constexpr size_t TW_BYTES = sizeof(TwT) * N;
    static constexpr size_t RING_OFF = (TW_BYTES + 127) & ~size_t(127);
    static constexpr size_t RING_BYTES = CHUNK_BYTES * G * PC;
    static constexpr size_t TILE_OFF = RING_OFF + RING_BYTES;
    static constexpr size_t TILE_ROWS = size_t(G) * B;
    static constexpr size_t TILE_BYTES = sizeof(float2) * TILE_ROWS * STRIDE;
    // FFT pass groups: one per warpgroup where the tile's rows split evenly
    static constexpr bool FFT_SPLIT = TILE_ROWS % FFT_WG_ == 0;
    static constexpr int PNT = FFT_SPLIT ? 128 : NFFT;  // threads per pass group
    static constexpr int PROWS = FFT_SPLIT ? int(TILE_ROWS) / FFT_WG_ : int(TILE_ROWS);
    static constexpr int PGROUPS = FFT_SPLIT ? FFT_WG_ : 1;
    // detection (POWER): last-pass units per row; a thread's units all have
    // the same bins when PNT is a multiple of it, so its FP64 accumulators
    // stay per bin — partial rows per CTA: PNT / UL per pass group
    static constexpr int UL = N >> FftSchedule<L - RLOG, W>::width(FftSchedule<L - RLOG, W>::NP - 1);
    static constexpr bool POWER_OK = T > 1 && PNT % UL == 0;
    static constexpr int POWER_ROWS = PGROUPS * (PNT / UL);
    static constexpr size_t BAR_OFF = (TILE_OFF + NTILE * TILE_BYTES + 7) & ~size_t(7);
    static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) * 2 * G * PC;
    static_assert(NTG >= 32 && NTG <= NFIR && NFIR % NTG == 0, "FIR groups must be whole warps");
    // setmaxnreg moves registers within the CTA's launch allocation only: the
    // split must fit (65536 / NT) rounded down to 8, or .inc waits forever
    static constexpr int LAUNCH_REGS = (65536 / NT) & ~7;
    static_assert(FIR_REGS * NFIR + FFT_REGS * NFFT <= LAUNCH_REGS * NT, "register split");
    static_assert(SMEM <= 232448, "shared memory per CTA");
    static_assert(BU * B <= 32, "FIR unroll too large");
    static_assert(!HS || FFT_SPLIT, "per-pass-group handoff needs an evenly split tile");
    static_assert(!HS || 1 + 2 * NTILE * PGROUPS + PGROUPS <= 16, "named barriers");
    static_assert(!TRIV || (!EXACT && RLOG >= 1 && RLOG <= 2), "trivial prestages: FAST, R = 2 or 4");
    static_assert(!PAIR || (B % 2 == 0 && T >= 2 && (!HS || PROWS % 2 == 0)),
                  "spectrum pairs within a batch and a pass group");
    // named barrier ids (0 = __syncthreads): FULL[t][pg], EMPTY[t][pg], pass
    // syncs per pass group (HS: per pass group; else one FULL / EMPTY per tile)
    static constexpr int HPG = HS ? PGROUPS : 1;          // handoff groups per tile
    // threads on pass group pg's handoff barriers: the FIR groups writing any
    // of its rows [pg*PROWS, (pg+1)*PROWS) (group g writes rows g*B .. g*B+B-1)
    // and the pass group's own threads; the whole CTA without HS
    PPFG_HD static constexpr int hcount(int pg) {
        return HS ? NTG * (((pg + 1) * PROWS - 1) / B - (pg * PROWS) / B + 1) + PNT : NT;
    }
    PPFG_HD static constexpr int bar_full(int t, int pg) { return 1 + t * HPG + pg; }
    PPFG_HD static constexpr int bar_empty(int t, int pg) { return 1 + NTILE * HPG + t * HPG + pg; }
    PPFG_HD static constexpr int bar_pass(int pg) { return 1 + 2 * NTILE * HPG + pg; }
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

// Tile row r of an FFT warpgroup that owns rows [off, off + rows): map its
// local row index to the tile's output rows.
struct OffsetRows {
    FusedRows base;
    int off;
    PPFG_DEV long long operator()(int r) const { return base(r + off); }
};

// named barriers: 0 = __syncthreads, FULL = 1+t, EMPTY = 1+NTILE+t, FFT
// passes = 1+2*NTILE + warpgroup (rows are independent: each FFT warpgroup
// transforms its own rows of the tile and syncs only with itself between
// passes)
PPFG_DEV void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
PPFG_DEV void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
struct SyncNamed {
    int id, count;
    PPFG_DEV void operator()() const { named_sync(id, count); }
};

PPFG_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// POWER = true: the detection variant (cli.hpp:307-317 fused into the final
// FFT pass): no bins are written; each FFT thread accumulates the powers of
// the bins it owns over all of the CTA's spectra and `out` receives per-CTA
// partial sums, double[gridDim.x][TILE_ROWS][N] (reduced by power_reduce_kernel).
template <class Cfg, bool POWER = false>
__global__ void __launch_bounds__(Cfg::NT, 1)
    fused_fir_fft_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                         long long S_out, long long rows_per_cta, const float* __restrict__ taps,
                         const typename Cfg::TwT* __restrict__ tw_g) {
    constexpr int L = Cfg::L, T = Cfg::T, RLOG = Cfg::RLOG, N = Cfg::N, R = Cfg::R;
    constexpr int NTG = Cfg::NTG, NFIR = Cfg::NFIR, NT = Cfg::NT;
    constexpr int G = Cfg::G, B = Cfg::B;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    typename Cfg::TwT* tw = reinterpret_cast<typename Cfg::TwT*>(smem_raw);
    float2* ring = reinterpret_cast<float2*>(smem_raw + Cfg::RING_OFF);
    float2* tiles = reinterpret_cast<float2*>(smem_raw + Cfg::TILE_OFF);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + Cfg::BAR_OFF);
    uint64_t* empty = full + G * Cfg::PC;

    const int tid = threadIdx.x;
    const long long o0 = static_cast<long long>(blockIdx.x) * rows_per_cta;
    const long long o1 = min(o0 + rows_per_cta, S_out);
    const long long rows_cta = max(o1 - o0, 0LL);
    const long long rpg = (rows_cta + G - 1) / G;
    // rounded up to whole FIR unrolls (BU batches): trailing batches are all
    // padding rows, computed and never stored, so the FIR body has no exits
    const long long n_batches = ((rpg + B - 1) / B + Cfg::BU - 1) / Cfg::BU * Cfg::BU;

    for (int i = tid; i < N - 1; i += NT)
        tw[i] = tw_g[i];
    if (tid < G * Cfg::PC) {
        mbar_init(full + tid, 1);
        mbar_init(empty + tid, Cfg::FW);
    }
    fence_mbar_init();
    __syncthreads();

    if (tid >= NFIR) {
        // ================================ FFT role ================================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::FFT_REGS));
        const int ftid = tid - NFIR;
        // per-warpgroup rows where the tile splits evenly, else CTA-wide passes
        constexpr bool SPLIT = Cfg::FFT_SPLIT;
        constexpr int PNT = Cfg::PNT, PROWS = Cfg::PROWS;
        const int pg = SPLIT ? ftid / 128 : 0;                  // pass group
        const int ptid = ftid - pg * PNT;
        using Passes = FftPasses<L, L - RLOG, Cfg::W, false, true, PNT, 0, true, POWER>;
        constexpr int EL = Passes::E_LAST;
        // detection accumulators: FP64 in EXACT mode (cmd_inspect's double
        // running sum up to order); FP32 in FAST mode, flushed into the CTA's
        // FP64 partial row every kFlush batches (fewer registers, no FP64 /
        // conversion work per bin; adds <= kFlush FP32 roundings per partial)
        using PA = typename std::conditional<Cfg::EXACT, double, float>::type;
        constexpr long long kFlush = 16;
        PA pacc[POWER ? EL : 1];
#pragma unroll
        for (int k = 0; k < (POWER ? EL : 1); ++k)
            pacc[k] = 0;
        double* part = nullptr;
        if constexpr (POWER) {
            // every last-pass unit of this thread (tile rows ptid / UL +
            // m * PNT / UL) covers bins u + rev_L(k): partial row r of the CTA
            constexpr int UL = N / EL;
            static_assert(UL == Cfg::UL && Cfg::POWER_OK, "per-bin accumulators");
            const int r = pg * (PNT / UL) + ptid / UL;
            const unsigned u = static_cast<unsigned>(ptid % UL);
            part = reinterpret_cast<double*>(out) +
                   (static_cast<size_t>(blockIdx.x) * Cfg::POWER_ROWS + r) * N + u;
        }
        bool flushed = false; // the partial row holds a value (else: store, not add)
        auto flush = [&]() {
#pragma unroll
            for (int k = 0; k < EL; ++k) {
                double* d = part + crev(static_cast<unsigned>(k), L);
                *d = (flushed ? *d : 0.0) + static_cast<double>(pacc[k]);
                pacc[k] = 0;
            }
            flushed = true;
        };
        const int hpg = Cfg::HS ? pg : 0;
        for (long long b = 0; b < n_batches; ++b) {
            const int t = static_cast<int>(b % Cfg::NTILE);
            named_sync(Cfg::bar_full(t, hpg), Cfg::hcount(hpg));
            Passes::run(nullptr, out,
                        tiles + (t * Cfg::TILE_ROWS + pg * PROWS) * Cfg::STRIDE, Cfg::STRIDE,
                        PROWS, OffsetRows{FusedRows{o0, o1, rpg, b * B, B}, pg * PROWS}, tw, ptid,
                        SyncNamed{Cfg::bar_pass(pg), PNT}, pacc);
            named_arrive(Cfg::bar_empty(t, hpg), Cfg::hcount(hpg));
            if constexpr (POWER && !Cfg::EXACT) {
                if ((b + 1) % kFlush == 0)
                    flush();
            }
        }
        if constexpr (POWER)
            flush();
        return;
    }

    // ================================== FIR role ==================================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::FIR_REGS));
    using Acc = typename std::conditional<Cfg::EXACT, double, float>::type;
    using Win = typename std::conditional<Cfg::EXACT, double2, float2>::type;
    constexpr int PC = Cfg::PC, BU = Cfg::BU;
    const int g = tid / NTG;
    const int j = tid - g * NTG;
    const bool producer = (j == 0);
    const bool warp_leader = (tid & 31) == 0;
    const long long og0 = o0 + g * rpg;
    const long long og1 = min(og0 + rpg, o1);
    const long long n_out_g = max(og1 - og0, 0LL);
    const long long n_chunks = (n_out_g + B - 1) / B; // chunk c = outputs cB..cB+B-1
    const float2* gsrc = in + og0 * N; // group input spectrum q = og0 + q
    float2* ring_g = ring + static_cast<size_t>(g) * PC * B * N;
    uint64_t* full_g = full + g * PC;
    uint64_t* empty_g = empty + g * PC;

    // chunk c = input spectra [T-1 + cB, T-1 + cB + B): the inputs batch c needs
    auto issue = [&](long long c) {
        const int slot = static_cast<int>(c % PC);
        const long long rows = min(static_cast<long long>(B), n_out_g - c * B);
        const uint32_t bytes = static_cast<uint32_t>(rows * N * sizeof(float2));
        mbar_arrive_expect_tx(full_g + slot, bytes);
        bulk_g2s(ring_g + static_cast<size_t>(slot) * B * N, gsrc + (T - 1 + c * B) * N, bytes,
                 full_g + slot);
        // warm L2 with the chunks after the ring's depth (no shared memory
        // needed): their bulk copies then start from L2
        if constexpr (Cfg::L2A > 0) {
            const long long cp = c + Cfg::L2A;
            if (cp < n_chunks) {
                const long long rp = min(static_cast<long long>(B), n_out_g - cp * B);
                bulk_prefetch_l2(gsrc + (T - 1 + cp * B) * N, static_cast<uint32_t>(rp * N * sizeof(float2)));
            }
        }
    };
    if (producer) {
        for (long long c = 0; c < n_chunks && c < PC; ++c)
            issue(c);
    }

    // taps and windows of channels c_k = j + k*NTG; window slots 1..T-1 hold
    // the T-1 warm-up spectra (read straight from global: once per group)
    Acc h[R][T];
    Win xw[R][T];
#pragma unroll
    for (int k = 0; k < R; ++k) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
            h[k][t] = static_cast<Acc>(__ldg(taps + static_cast<size_t>(t) * N + j + k * NTG));
            float2 x = make_float2(0.f, 0.f);
            if (t >= 1 && n_out_g > 0)
                x = __ldg(gsrc + static_cast<long long>(t - 1) * N + j + k * NTG);
            xw[k][t].x = static_cast<Acc>(x.x);
            xw[k][t].y = static_cast<Acc>(x.y);
        }
    }
    // pre-stage twiddles tw[0 .. R-2] are the same for every spectrum
    float4 twr[R > 1 ? R - 1 : 1];
#pragma unroll
    for (int i = 0; i + 1 < R; ++i)
        twr[i] = tw_load<true>(tw + i);

    const unsigned swj = sw(static_cast<unsigned>(j));
    for (long long b0 = 0; b0 < n_batches; b0 += BU) {
#pragma unroll
        for (int u = 0; u < BU; ++u) {
            const long long b = b0 + u;
            const int t = static_cast<int>(b % Cfg::NTILE);
            const int slot = static_cast<int>(b % PC);
            const bool have = b < n_chunks;
            if (producer && b >= 1 && b - 1 + PC < n_chunks) {
                // refill the slot batch b-1 released
                mbar_wait(empty_g + (b - 1) % PC, static_cast<uint32_t>(((b - 1) / PC) & 1));
                fence_proxy_async();
                issue(b - 1 + PC);
            }
            if (!Cfg::HS && b >= Cfg::NTILE)
                named_sync(Cfg::bar_empty(t, 0), NT); // the FFT role has drained tile t
            if (have)
                mbar_wait(full_g + slot, static_cast<uint32_t>((b / PC) & 1));
            const float2* chunk = ring_g + static_cast<size_t>(slot) * B * N + j;
            float2* tile = tiles + t * Cfg::TILE_ROWS * Cfg::STRIDE + g * B * Cfg::STRIDE + swj;
            // Rows past the group's end (partial or absent chunk) read stale
            // ring data: they only feed outputs the FFT role never stores, and
            // keeping the loads unpredicated lets the window rotate by renaming.
            if constexpr (Cfg::PAIR) {
#pragma unroll
                for (int i = 0; i < B; i += 2) {
                    if constexpr (Cfg::HS) { // tile rows g*B+i, +1: their pass group has drained tile t
                        const int r = g * B + i;
                        if ((i == 0 || r % Cfg::PROWS == 0) && b >= Cfg::NTILE)
                            named_sync(Cfg::bar_empty(t, r / Cfg::PROWS), Cfg::hcount(r / Cfg::PROWS));
                    }
                    float2 y0[R], y1[R];
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        // window: xw[k][t] = x[i + t - 1], t = 1..T-1; output i reads
                        // (xw[1..T-1], a), output i+1 (xw[2..T-1], a, b)
                        const float2 xa = chunk[i * N + k * NTG], xb = chunk[(i + 1) * N + k * NTG];
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
                        fft_prestages<L, RLOG>(y0, twr);
                        fft_prestages<L, RLOG>(y1, twr);
                    }
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        tile[i * Cfg::STRIDE + sw(static_cast<unsigned>(k * NTG))] = y0[k];
                        tile[(i + 1) * Cfg::STRIDE + sw(static_cast<unsigned>(k * NTG))] = y1[k];
                    }
                    if constexpr (Cfg::HS) { // this group's rows of the pass group are written
                        const int r = g * B + i + 1;
                        if (i + 1 == B - 1 || (r + 1) % Cfg::PROWS == 0)
                            named_arrive(Cfg::bar_full(t, r / Cfg::PROWS), Cfg::hcount(r / Cfg::PROWS));
                    }
                }
            } else {
    #pragma unroll
                for (int i = 0; i < B; ++i) {
                    if constexpr (Cfg::HS) { // tile row g*B+i's pass group has drained tile t
                        const int r = g * B + i;
                        if ((i == 0 || r % Cfg::PROWS == 0) && b >= Cfg::NTILE)
                            named_sync(Cfg::bar_empty(t, r / Cfg::PROWS), Cfg::hcount(r / Cfg::PROWS));
                    }
                    float2 y[R];
    #pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const float2 x = chunk[i * N + k * NTG];
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
                        fft_prestages<L, RLOG>(y, twr);
    #pragma unroll
                    for (int k = 0; k < R; ++k)
                        tile[i * Cfg::STRIDE + sw(static_cast<unsigned>(k * NTG))] = y[k];
                    if constexpr (Cfg::HS) { // this group's rows of the pass group are written
                        const int r = g * B + i;
                        if (i == B - 1 || (r + 1) % Cfg::PROWS == 0)
                            named_arrive(Cfg::bar_full(t, r / Cfg::PROWS), Cfg::hcount(r / Cfg::PROWS));
                    }
                }
            }
            __syncwarp();
            if (have && warp_leader)
                mbar_arrive(empty_g + slot); // this warp is done with the chunk
            if constexpr (!Cfg::HS)
                named_arrive(Cfg::bar_full(t, 0), NT); // tile t is full
        }
    }
}

// Per-channel mean power from per-CTA partials: mean[c] = (sum over parts,
// in a fixed order) / n — deterministic for a given grid.
static __global__ void power_reduce_kernel(const double* __restrict__ part, int n_parts, int C,
                                    double n, double* __restrict__ mean) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C)
        return;
    double s = 0.0;
    for (int i = 0; i < n_parts; ++i)
        s += part[static_cast<size_t>(i) * C + c];
    mean[c] = n > 0 ? s / n : 0.0;
}

// cmd_inspect on channelized bins (cli.hpp:307-317): CTA g sums the powers of
// spectra [g*rows_per_cta, ...) per channel (thread = channel stripe), in
// spectrum order, into part[g][c].
static __global__ void __launch_bounds__(256) power_partial_kernel(const float2* __restrict__ bins,
                                                            long long n_spectra, int C,
                                                            long long rows_per_cta,
                                                            double* __restrict__ part) {
    const long long s0 = static_cast<long long>(blockIdx.x) * rows_per_cta;
    const long long s1 = min(s0 + rows_per_cta, n_spectra);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        double acc = 0.0;
        const float2* p = bins + s0 * C + c;
        long long s = s0;
        for (; s + 8 <= s1; s += 8, p += 8 * static_cast<long long>(C)) {
            float2 a[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                a[i] = __ldcs(p + i * static_cast<long long>(C));
#pragma unroll
            for (int i = 0; i < 8; ++i)
                acc += static_cast<double>(a[i].x) * a[i].x + static_cast<double>(a[i].y) * a[i].y;
        }
        for (; s < s1; ++s, p += C) {
            const float2 a = __ldcs(p);
            acc += static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y;
        }
        part[static_cast<size_t>(blockIdx.x) * C + c] = acc;
    }
}

} // namespace ppfg
