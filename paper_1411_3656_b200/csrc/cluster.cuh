// cluster.cuh — thread-block-cluster primitives used by the split kernel
// (fused_split.cuh): CTA rank, DSMEM address mapping, the remote mbarrier
// arrive, the cluster barrier, and the debug phase trace.
#pragma once

#include "fused.cuh"

namespace ppfg {

PPFG_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cta address -> the same offset in CTA `rank`'s shared memory
PPFG_DEV uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_addr), "r"(rank));
    return out;
}

// "I have finished reading this tile": the reads completed when their values
// were consumed (stored to HBM) before the named barrier that precedes this
// arrive, so it needs no release semantics — a release arrive would make the
// thread wait for all its outstanding HBM stores first.
PPFG_DEV void mbar_arrive_remote_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}

PPFG_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

#ifdef PPFG_TRACE
// debug builds only (-DPPFG_TRACE, scripts/build_trace.sh): %globaltimer
// stamps of CTA 0's phases, read back with ppfg_debug_trace
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

} // namespace ppfg
