// common.cuh — shared device helpers for the sm_100a PPF kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define PPFG_DEV __device__ __forceinline__
#define PPFG_HD __host__ __device__ __forceinline__

namespace ppfg {

// ---- compile-time bit helpers -------------------------------------------------
PPFG_HD constexpr unsigned crev(unsigned x, int nbits) {
    unsigned r = 0;
    for (int i = 0; i < nbits; ++i)
        r |= ((x >> i) & 1u) << (nbits - 1 - i);
    return r;
}

// runtime reverse of the low nbits (nbits >= 1)
PPFG_DEV unsigned crev_rt(unsigned x, int nbits) { return __brev(x) >> (32 - nbits); }

// Shared-memory swizzle for float2 rows: base-16 digit sum. Additive over
// disjoint bit sets (so sw(fixed | k<<LO) = sw(fixed) + sw(k<<LO), giving
// immediate-offset LDS/STS), and conflict-free whenever the 16 lanes of a
// half-warp vary any 4 consecutive label bits (their contributions mod 16 are
// 4 distinct powers of two).
PPFG_HD constexpr unsigned sw(unsigned n) { return n + (n >> 4) + (n >> 8) + (n >> 12); }
PPFG_HD constexpr unsigned sw_row_stride(unsigned N) { return ((sw(N - 1) + 1) + 1) & ~1u; }

// ---- the reference's radix-2 butterfly (dft.hpp:122-131), exact -------------
// tr = fma(br, wr, -(bi*wi)); ti = fma(br, wi, bi*wr); hi = lo - t; lo += t.
// The _rn intrinsics forbid contraction so every operation rounds exactly as
// the reference's explicit std::fma / float ops do.
PPFG_DEV void bfly(float2& lo, float2& hi, const float2 w) {
    const float br = hi.x, bi = hi.y;
    const float tr = __fmaf_rn(br, w.x, -__fmul_rn(bi, w.y));
    const float ti = __fmaf_rn(br, w.y, __fmul_rn(bi, w.x));
    hi.x = __fsub_rn(lo.x, tr);
    hi.y = __fsub_rn(lo.y, ti);
    lo.x = __fadd_rn(lo.x, tr);
    lo.y = __fadd_rn(lo.y, ti);
}

// ---- packed FP32x2 (sm_100a FFMA2/FMUL2/FADD2) --------------------------------------
// Each lane of a .f32x2 op rounds exactly like the scalar op, so these are
// bit-identical to the scalar reference arithmetic at half the instructions.
// A pair whose two halves are the same scalar compiles to the broadcast
// operand form (R.F32), so "scalar x pair" costs no extra move.
PPFG_DEV unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
PPFG_DEV float2 upk2(unsigned long long r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
PPFG_DEV float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(d)
        : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
    return upk2(d);
}
PPFG_DEV float2 mul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(d);
}
PPFG_DEV float2 add2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(d);
}
PPFG_DEV float2 sub2(float2 a, float2 b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
    return upk2(d);
}
// scalar s times pair b (+ c)
PPFG_DEV float2 fma2s(float s, float2 b, float2 c) { return fma2(make_float2(s, s), b, c); }
PPFG_DEV float2 mul2s(float s, float2 b) { return mul2(make_float2(s, s), b); }

// The same butterfly on packed pairs with w4 = (wr, wi, -wi, wr):
//   m = bi * (-wi, wr)            -> (-(bi*wi), bi*wr)    [RN each lane]
//   t = br * (wr, wi) + m         -> (fma(br,wr,-(bi*wi)), fma(br,wi,bi*wr))
//   hi = lo - t; lo = lo + t
// 4 packed instructions (FMUL2, FFMA2, 2x FADD2) for the reference's 8.
// Twiddles live in memory as float2 (wr, wi) — the reference's f32 table
// entry — and are expanded in registers to the (wr, wi, -wi, wr) operand
// bfly2 consumes: one MOV and one sign-bit LOP3 (exact negation) per twiddle,
// off the FMA pipe, for half the shared-memory bytes of a stored float4.
PPFG_DEV float4 tw_expand(float2 w) {
    uint32_t nwi;
    asm("xor.b32 %0, %1, 0x80000000;" : "=r"(nwi) : "r"(__float_as_uint(w.y)));
    return make_float4(w.x, w.y, __uint_as_float(nwi), w.x);
}

PPFG_DEV void bfly2(float2& lo, float2& hi, const float4 w) {
    const float2 m = mul2s(hi.y, make_float2(w.z, w.w));
    const float2 t = fma2s(hi.x, make_float2(w.x, w.y), m);
    hi = sub2(lo, t);
    lo = add2(lo, t);
}

// ---- mbarrier / bulk-copy (TMA 1-D) PTX wrappers --------------------------------
PPFG_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

PPFG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

PPFG_DEV void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

PPFG_DEV void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

PPFG_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

PPFG_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// non-blocking probe of a phase (mbarrier.test_wait never suspends)
PPFG_DEV bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

PPFG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// global -> shared bulk copy completing on an mbarrier (SASS: UBLKCP).
// bytes % 16 == 0, both addresses 16-byte aligned.
PPFG_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a global range (cp.async.bulk.prefetch.L2; no shared memory,
// no completion tracking): warms L2 for a later bulk copy of the same bytes
PPFG_DEV void bulk_prefetch_l2(const void* gmem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem_src), "r"(bytes) : "memory");
}

// streaming (evict-first) 8-byte global store
PPFG_DEV void st_cs(float2* p, float2 v) { __stcs(p, v); }

} // namespace ppfg
