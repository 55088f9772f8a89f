// fused_cluster.cuh — K3c: the fused FIR+FFT for channel/tap counts whose
// FIR state does not fit one SM's register file (C >= 2048, T >= 16, FP64 at
// C = 1024): a thread-block cluster of Q = 2^LQ CTAs (one per SM) works on
// the same output spectra, CTA r owning channels n = Q*m + r.
//
// Why this split: in the reference's radix-2 DIT (labels n = channel index,
// stage s pairs labels differing in bit L-s), every stage but the last LQ
// pairs labels with equal low bits, and those stages on the decimated
// sequence x[Q*m + r] use exactly the twiddles tw[h-1+j] of an (N/Q)-point
// transform. So each CTA runs the single-SM machinery of fused.cuh for
// N_loc = N/Q on its own channels, and only the last LQ stages combine the Q
// sub-transforms. Local label m with low bits d belongs to the cross group
// handled by CTA d: in its last local pass every CTA PUSHES each value
// straight into the owner's inbox over DSMEM (st.shared::cluster, fire and
// forget), so the cross stages read only local shared memory. The owner runs
// the LQ stages in registers with the reference twiddles and stores the Q
// bins rev(r')*N/Q + rev(rank)*N/Q^2 + u (coalesced runs).
//
// Input: CTA r's channels are strided by Q, which TMA cannot express (no
// element stride on the innermost dimension, 16-byte minimum box row), so
// each FIR thread streams its own channels through a private D-row ring in
// shared memory with cp.async (LDGSTS) — no cross-thread handshakes, D rows
// of every thread in flight.
//
// Synchronisation per tile t (two tiles and two inboxes):
//   FIR -> FFT (same CTA)      : named barrier FULL[t]
//   FFT -> FIR (same CTA)      : named barrier EMPTY[t] once the local passes
//                                 have read the tile (the inbox holds the rest)
//   pushes into inboxes landed : one arrive per CTA on every CTA's ready[t]
//                                 (release.cluster after a cluster fence)
//   inbox t read by its owner  : one arrive per CTA on every CTA's free[t];
//                                 a CTA waits on its own free[t] before pushing
//                                 into anyone's inbox t again.
#pragma once

#include "fused.cuh"

namespace ppfg {

PPFG_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
PPFG_DEV uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_addr), "r"(rank));
    return out;
}
PPFG_DEV float2 ld_cluster_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr)
                 : "memory");
    return v;
}
// Remote arrive / local wait with the default (CTA-scope release/acquire)
// semantics, as CUTLASS's cluster pipelines use them: the exchanged data lives
// in shared memory, read over DSMEM straight from the owner SM, so no L1
// invalidation is needed — a cluster-scope acquire would emit CCTL.IVALL on
// every poll.
PPFG_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// poll with CTA-scope acquire, then one cluster-scope fence (CCTL once per
// wait instead of once per poll)
PPFG_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    mbar_wait(bar, parity);
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
}
// "I have read my inbox": the inbox values were consumed (stored to HBM)
// before the named barrier that precedes this arrive, so no fence is needed; a
// release arrive here would make thread 0 wait for all its HBM stores.
PPFG_DEV void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
PPFG_DEV void st_cluster_f2(uint32_t addr, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y)
                 : "memory");
}
// remote store that completes its bytes on the target CTA's mbarrier
PPFG_DEV void st_async_f2(uint32_t addr, float2 v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "f"(v.x), "f"(v.y), "r"(mbar)
                 : "memory");
}
PPFG_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
PPFG_DEV float2 ldg_na_f2(const float2* p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y)
                 : "l"(p));
    return v;
}
PPFG_DEV void cp_async8(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
                 : "memory");
}
PPFG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
PPFG_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#ifdef PPFG_TRACE
// debug builds only (-DPPFG_TRACE): %globaltimer stamps of CTA 0's phases,
// read back with ppfg_debug_trace
__device__ unsigned long long g_trace[2][16][64];
PPFG_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PPFG_TR(role, b, ev)                                                                      \
    do {                                                                                          \
        if (blockIdx.x == 0 && (b) < 64)                                                          \
            g_trace[role][ev][b] = gtimer();                                                      \
    } while (0)
#else
#define PPFG_TR(role, b, ev)                                                                      \
    do {                                                                                          \
    } while (0)
#endif

template <int L_, int LQ_, int T_, int RLOG_, bool EXACT_, int FIR_REGS_ = 160, int FFT_REGS_ = 96>
struct ClusterCfg {
    static constexpr int L = L_, LQ = LQ_, T = T_, RLOG = RLOG_;
    static constexpr bool EXACT = EXACT_;
    static constexpr int FIR_REGS = FIR_REGS_, FFT_REGS = FFT_REGS_;
    static constexpr int Q = 1 << LQ;
    static constexpr int N = 1 << L;
    static constexpr int LL = L - LQ;           // local label bits
    static constexpr int NL = 1 << LL;          // local channels per CTA
    static constexpr int R = 1 << RLOG;
    static constexpr int NTG = NL / R;          // FIR threads per group
    static constexpr int NFIR = 256, NFFT = 256, NT = NFIR + NFFT;
    static constexpr int G = NFIR / NTG;
    static constexpr int W = 4;
    static constexpr int B = (NFFT << W) / (NL * G) > 0 ? (NFFT << W) / (NL * G) : 1;
    static constexpr int BU = ilcm(B, T) / B;
    static constexpr int PD = (R >= 4 || EXACT) ? 4 : 8; // register prefetch depth (spectra)
    static constexpr unsigned STRIDE = sw_row_stride(NL);
    // the whole table (cross stages too) when it fits, else the local part
    static constexpr bool TW_ALL = sizeof(float4) * N <= 80 * 1024;
    static constexpr size_t TW_BYTES = sizeof(float4) * (TW_ALL ? N : NL);
    static constexpr size_t TILE_OFF = (TW_BYTES + 127) & ~size_t(127);
    static constexpr size_t TILE_ROWS = size_t(G) * B;
    static constexpr size_t TILE_BYTES = sizeof(float2) * TILE_ROWS * STRIDE;
    // inbox: [tile][source CTA][row][sw(m >> LQ)] for the labels this CTA owns
    static constexpr unsigned IN_STRIDE = sw_row_stride(NL / Q);
    static constexpr size_t INBOX_OFF = TILE_OFF + 2 * TILE_BYTES;
    static constexpr size_t INBOX_TILE = sizeof(float2) * size_t(Q) * TILE_ROWS * IN_STRIDE;
    static constexpr size_t BAR_OFF = (INBOX_OFF + 2 * INBOX_TILE + 7) & ~size_t(7);
    static constexpr size_t SMEM = BAR_OFF + sizeof(uint64_t) * 4;
    static_assert(FftSchedule<LL - RLOG, W>::NP == 2, "local FFT = exactly two passes");
    static_assert(LQ >= 1 && LQ <= 3, "cluster of 2..8 CTAs");
    static_assert(LL >= LQ, "N/Q must be >= Q");
    static_assert(NTG >= 32 && NTG <= NFIR && NFIR % NTG == 0, "FIR groups must be whole warps");
    static constexpr int LAUNCH_REGS = (65536 / NT) & ~7;
    static_assert(FIR_REGS * NFIR + FFT_REGS * NFFT <= LAUNCH_REGS * NT, "register split");
    static_assert(SMEM <= 232448, "shared memory per CTA");
    static_assert((BU * B) % PD == 0, "prefetch slots must be compile-time in the FIR body");
    static_assert(PD <= T - 1 + B || true, "");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, 1)
    fused_cluster_kernel(const float2* __restrict__ in, float2* __restrict__ out, long long S_out,
                         long long rows_per_cluster, const float* __restrict__ taps,
                         const float4* __restrict__ tw_g) {
    constexpr int L = Cfg::L, LQ = Cfg::LQ, Q = Cfg::Q, N = Cfg::N, LL = Cfg::LL, NL = Cfg::NL;
    constexpr int T = Cfg::T, RLOG = Cfg::RLOG, R = Cfg::R, NTG = Cfg::NTG;
    constexpr int NFIR = Cfg::NFIR, NFFT = Cfg::NFFT, NT = Cfg::NT, G = Cfg::G, B = Cfg::B;
    constexpr int PD = Cfg::PD, BU = Cfg::BU;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float4* tw = reinterpret_cast<float4*>(smem_raw);
    float2* tiles = reinterpret_cast<float2*>(smem_raw + Cfg::TILE_OFF);
    float2* inbox = reinterpret_cast<float2*>(smem_raw + Cfg::INBOX_OFF);
    uint64_t* ready = reinterpret_cast<uint64_t*>(smem_raw + Cfg::BAR_OFF);
    uint64_t* freed = ready + 2;

    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const long long cluster_id = blockIdx.x / Q;
    const long long o0 = cluster_id * rows_per_cluster;
    const long long o1 = min(o0 + rows_per_cluster, S_out);
    const long long rows_cta = max(o1 - o0, 0LL);
    const long long rpg = (rows_cta + G - 1) / G;
    const long long n_batches = ((rpg + B - 1) / B + BU - 1) / BU * BU;

    for (int i = tid; i < (Cfg::TW_ALL ? N : NL) - 1; i += NT)
        tw[i] = tw_g[i]; // local stages use tw[0 .. NL-2]; cross stages the rest
    const float4* tw_x = Cfg::TW_ALL ? tw : tw_g;
    if (tid < 2) {
        mbar_init(ready + tid, 1);  // own expect_tx arrive + the pushed bytes
        mbar_init(freed + tid, Q);  // one arrival per owner CTA
    }
    fence_mbar_init();
    __syncthreads();
    cluster_sync_all(); // every CTA's barriers exist before anyone arrives remotely

    if (tid >= NFIR) {
        // ================================ FFT role ================================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::FFT_REGS));
        using S = FftSchedule<LL - RLOG, Cfg::W>;
        constexpr int W1 = S::width(1);    // last local pass: label bits [0, W1)
        constexpr int U1 = NL >> W1;
        constexpr int UPR = NL / Q;        // cross-stage units per spectrum (Q bins each)
        constexpr int UPT = static_cast<int>(Cfg::TILE_ROWS) * UPR / NFFT;
        static_assert(static_cast<int>(Cfg::TILE_ROWS) * UPR % NFFT == 0, "cross units");
        static_assert(W1 >= LQ, "the owner CTA is a compile-time function of the lane's value");
        // bytes each CTA receives from the other Q-1 CTAs per tile (own values
        // are written locally)
        constexpr uint32_t PAYLOAD = sizeof(float2) * Cfg::TILE_ROWS * (NL / Q) * (Q - 1);
        const int ftid = tid - NFIR;
        const uint32_t inbox_addr = smem_u32(inbox);
        const uint32_t ready_addr = smem_u32(ready);
        // Software-pipelined: iteration b runs the local passes of tile b, then
        // the cross stages of tile b-1, so the partner CTAs' pushes for b-1
        // have a whole local-pass time to land before they are waited for.
        auto cross = [&](long long bp) {
            const int tp = static_cast<int>(bp & 1);
            const FusedRows map{o0, o1, rpg, bp * B, B};
            mbar_wait(ready + tp, static_cast<uint32_t>((bp >> 1) & 1));
            // unit u of row r -> local label m = rev(u) << LQ | rank; its Q values
            // sit in this CTA's inbox tp, one per source CTA
            if (ftid == 0) PPFG_TR(1, bp, 6);
            const float2* ib = inbox + tp * Q * Cfg::TILE_ROWS * Cfg::IN_STRIDE;
            float2 v[UPT][Q];
            unsigned mm[UPT];
#pragma unroll
            for (int i = 0; i < UPT; ++i) {
                const int unit = ftid + i * NFFT;
                const int r = unit / UPR;
                const unsigned u = static_cast<unsigned>(unit - r * UPR);
                const unsigned mp = (LL - LQ > 0) ? crev_rt(u, LL - LQ) : 0u;
                mm[i] = (mp << LQ) | rank;
#pragma unroll
                for (int r2 = 0; r2 < Q; ++r2)
                    v[i][r2] = ib[(r2 * Cfg::TILE_ROWS + r) * Cfg::IN_STRIDE + sw(mp)];
            }
#pragma unroll
            for (int i = 0; i < UPT; ++i) {
                const unsigned m = mm[i];
#pragma unroll
                for (int bb = LQ - 1; bb >= 0; --bb) {
                    const int s = L - bb;
                    const unsigned half = 1u << (s - 1);
#pragma unroll
                    for (int r2 = 0; r2 < Q; ++r2) {
                        if (r2 & (1 << bb))
                            continue;
                        const unsigned n = (m << LQ) | static_cast<unsigned>(r2);
                        const unsigned j = __brev(n >> (bb + 1)) >> (33 - s);
                        bfly2(v[i][r2], v[i][r2 | (1 << bb)], tw_x[half - 1 + j]);
                    }
                }
                const int unit = ftid + i * NFFT;
                const int r = unit / UPR;
                const unsigned u = static_cast<unsigned>(unit - r * UPR);
                const long long grow = map(r);
                if (grow >= 0) {
                    float2* dst = out + grow * N + crev(rank, LQ) * (NL / Q) + u;
#pragma unroll
                    for (int r2 = 0; r2 < Q; ++r2)
                        st_cs(dst + crev(static_cast<unsigned>(r2), LQ) * NL, v[i][r2]);
                }
            }
            named_sync(5, NFFT);
            if (ftid == 0) { // inbox tp is read: its writers may push into it again
#pragma unroll
                for (int r2 = 0; r2 < Q; ++r2)
                    mbar_arrive_remote_relaxed(mapa(smem_u32(freed + tp), r2));
            }
        };
        for (long long b = 0; b < n_batches; ++b) {
            const int t = static_cast<int>(b & 1);
            float2* tile = tiles + t * Cfg::TILE_ROWS * Cfg::STRIDE;
            const FusedRows map{o0, o1, rpg, b * B, B};
            if (ftid == 0)
                mbar_arrive_expect_tx(ready + t, PAYLOAD);
            if (ftid == 0) PPFG_TR(1, b, 0);
            named_sync(1 + t, NT);
            if (ftid == 0) PPFG_TR(1, b, 1);
            // local pass 0 (label bits [W1, LL-RLOG)), back into the tile
            fft_tile_pass<LL, S::lo(0), S::width(0), false, false, true, NFFT>(
                nullptr, nullptr, tile, Cfg::STRIDE, static_cast<int>(Cfg::TILE_ROWS), map, tw,
                ftid);
            named_sync(5, NFFT);
            if (ftid == 0) PPFG_TR(1, b, 2);
            if (b >= 2) // every owner has read its inbox t from batch b-2
                mbar_wait(freed + t, static_cast<uint32_t>(((b >> 1) - 1) & 1));
            if (ftid == 0) PPFG_TR(1, b, 3);
            // local pass 1 (label bits [0, W1)); each value goes to the inbox of the
            // CTA owning its cross group (label low bits): st.async completing bytes
            // on that CTA's ready[t], or a plain store for this CTA's own group
            for (int unit = ftid; unit < static_cast<int>(Cfg::TILE_ROWS) * U1; unit += NFFT) {
                const int r = unit / U1;
                const unsigned u = static_cast<unsigned>(unit - r * U1);
                const unsigned fixed = crev_rt(u, LL - W1) << W1;
                float2 v[1 << W1];
                const float2* src = tile + r * Cfg::STRIDE + sw(fixed);
#pragma unroll
                for (int k = 0; k < (1 << W1); ++k)
                    v[k] = src[sw(static_cast<unsigned>(k))];
                fft_stages<LL, 0, W1, true>(v, fixed, tw);
                const uint32_t slot0 =
                    inbox_addr + static_cast<uint32_t>(
                                     ((t * Q + static_cast<int>(rank)) * Cfg::TILE_ROWS + r) *
                                         Cfg::IN_STRIDE + sw(fixed >> LQ)) * sizeof(float2);
#pragma unroll
                for (int k = 0; k < (1 << W1); ++k) {
                    const uint32_t dest = static_cast<uint32_t>(k & (Q - 1));
                    const uint32_t a = slot0 + sw(static_cast<unsigned>(k) >> LQ) * sizeof(float2);
                    if (dest == rank)
                        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v[k].x),
                                     "f"(v[k].y)
                                     : "memory");
                    else
                        st_async_f2(mapa(a, dest), v[k], mapa(ready_addr + t * 8, dest));
                }
            }
            if (ftid == 0) PPFG_TR(1, b, 4);
            named_arrive(3 + t, NT); // tile t may be refilled by the FIR role
            named_sync(5, NFFT);     // own-group values visible to every FFT thread
            if (b >= 1)
                cross(b - 1);
            if (ftid == 0) PPFG_TR(1, b, 5);
        }
        if (n_batches >= 1)
            cross(n_batches - 1);
    } else {
        // ================================ FIR role ================================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::FIR_REGS));
        using Acc = typename std::conditional<Cfg::EXACT, double, float>::type;
        using Win = typename std::conditional<Cfg::EXACT, double2, float2>::type;
        const int g = tid / NTG;
        const int j = tid - g * NTG;
        const long long og0 = o0 + g * rpg;
        const long long og1 = min(og0 + rpg, o1);
        const long long n_out_g = max(og1 - og0, 0LL);
        const long long n_in_g = n_out_g > 0 ? n_out_g + T - 1 : 0;
        // this thread's channels: local labels j + k*NTG -> n = Q*m + rank. They are
        // strided by Q (no TMA box can express that), so each thread streams them
        // itself with non-L1-allocating loads, PD spectra ahead in registers (the
        // ~14 KB of L1 left beside 200+ KB of shared memory cannot stage them).
        const float2* src0 = in + og0 * N + static_cast<long long>(Q) * j + rank;
        float2 pf[PD][R];
        auto load_row = [&](long long q, float2 (&dst)[R]) {
            const long long qc = n_in_g > 0 ? min(q, n_in_g - 1) : 0; // clamped: unstored outputs
#pragma unroll
            for (int k = 0; k < R; ++k)
                dst[k] = ldg_na_f2(src0 + qc * N + static_cast<long long>(Q) * k * NTG);
        };
#pragma unroll
        for (int q = 0; q < PD; ++q)
            load_row(q, pf[q]);

        Acc h[R][T];
        Win xw[R][T];
#pragma unroll
        for (int k = 0; k < R; ++k) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
                h[k][t] = static_cast<Acc>(
                    __ldg(taps + static_cast<size_t>(t) * N + Q * (j + k * NTG) + rank));
                xw[k][t].x = Acc(0);
                xw[k][t].y = Acc(0);
            }
        }
        // warm-up: inputs 0..T-2 fill window slots 1..T-1
#pragma unroll
        for (int q = 0; q + 1 < T; ++q) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                xw[k][q + 1].x = static_cast<Acc>(pf[q % PD][k].x);
                xw[k][q + 1].y = static_cast<Acc>(pf[q % PD][k].y);
            }
            load_row(q + PD, pf[q % PD]);
        }
        float4 twr[R > 1 ? R - 1 : 1];
#pragma unroll
        for (int i = 0; i + 1 < R; ++i)
            twr[i] = tw[i];
        const unsigned swj = sw(static_cast<unsigned>(j));
        for (long long b0 = 0; b0 < n_batches; b0 += BU) {
#pragma unroll
            for (int uu = 0; uu < BU; ++uu) {
                const long long b = b0 + uu;
                const int t = static_cast<int>(b & 1);
                if (tid == 0) PPFG_TR(0, b, 0);
                if (b >= 2) // this CTA's FFT role has read tile t (batch b-2)
                    named_sync(3 + t, NT);
                if (tid == 0) PPFG_TR(0, b, 1);
                float2* tile = tiles + t * Cfg::TILE_ROWS * Cfg::STRIDE + g * B * Cfg::STRIDE + swj;
#pragma unroll
                for (int i = 0; i < B; ++i) {
                    const long long q = b * B + i + T - 1;
                    constexpr int slot_base = 0; // b0 * B is a multiple of PD
                    const int slot = (slot_base + uu * B + i + T - 1) % PD; // compile-time
                    float2 x[R];
#pragma unroll
                    for (int k = 0; k < R; ++k)
                        x[k] = pf[slot][k];
                    load_row(q + PD, pf[slot]); // prefetch PD spectra ahead
                    float2 y[R];
#pragma unroll
                    for (int k = 0; k < R; ++k) {
#pragma unroll
                        for (int tt = 0; tt + 1 < T; ++tt)
                            xw[k][tt] = xw[k][tt + 1];
                        xw[k][T - 1].x = static_cast<Acc>(x[k].x);
                        xw[k][T - 1].y = static_cast<Acc>(x[k].y);
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
                    fft_prestages<LL, RLOG>(y, twr);
#pragma unroll
                    for (int k = 0; k < R; ++k)
                        tile[i * Cfg::STRIDE + sw(static_cast<unsigned>(k * NTG))] = y[k];
                }
                if (tid == 0) PPFG_TR(0, b, 2);
                named_arrive(1 + t, NT);
            }
        }
    }
    cluster_sync_all(); // no CTA leaves while a partner may still read its tiles
}

} // namespace ppfg
