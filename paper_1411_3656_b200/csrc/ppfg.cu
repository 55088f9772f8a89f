// ppfg.cu — libppfg.so: plans, kernel dispatch, the host-streamed pipeline,
// device-resident streaming state, multi-GPU sharding and the C-ABI of
// include/ppfg.h. Kernels live in fir.cuh (K1), fft.cuh (K2), fused.cuh (K3),
// fused_split.cuh (K3s, thread-block clusters), dft.cuh (K4 dft_naive,
// K5 synth).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <list>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ppfg.h"
#include "tables.h"

#include "dft.cuh"
#include "fft.cuh"
#include "fir.cuh"
#include "fused.cuh"
#include "fused_split.cuh"

namespace ppfg {
void copy_piece(void* dst, const void* src, size_t n); // hostcopy.cpp
}

namespace {

using namespace ppfg;

// ------------------------------------------------------------------ errors
thread_local std::string g_err;
thread_local uint64_t g_err_offset = 0;
std::atomic<uint64_t> g_launches{0};

int fail(int status, const std::string& msg) {
    g_err = msg;
    return status;
}

#define PPFG_CUDA(call)                                                                           \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(PPFG_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)

#define PPFG_TRY(expr)                                                                            \
    do {                                                                                          \
        int st_ = (expr);                                                                         \
        if (st_ != PPFG_OK)                                                                       \
            return st_;                                                                           \
    } while (0)

int check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(PPFG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    return PPFG_OK;
}

bool is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }
int ilog2(uint64_t n) {
    int l = 0;
    while ((uint64_t(1) << l) < n)
        ++l;
    return l;
}
uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// RAII device guard
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev)
            cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev)
            cudaSetDevice(prev);
    }
};

// -------------------------------------------------------- kernel tables
// (tables.h; the kernel instantiations are compiled in the tab_*.cu units)
const std::vector<L2xEntry>& l2x_entries() {
    static const std::vector<L2xEntry> t = l2x_table();
    return t;
}

const std::vector<FusedEntry>& fused_table() {
    static const std::vector<FusedEntry> t = [] {
        std::vector<FusedEntry> v;
        for (auto part : {fused_part_main, fused_part_small, fused_part_fft, fused_part_split}) {
            auto p = part();
            v.insert(v.end(), p.begin(), p.end());
        }
        return v;
    }();
    return t;
}

// one-time per (device, function) opt-in to large dynamic shared memory
int ensure_smem_attr(KernelFn fn, size_t smem, int device) {
    static std::mutex mu;
    static std::map<std::pair<int, KernelFn>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(device, fn);
    auto it = done.find(key);
    if (it != done.end() && it->second >= smem)
        return PPFG_OK;
    if (smem > 48 * 1024)
        PPFG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
    done[key] = smem;
    return PPFG_OK;
}

} // namespace

// Pinned / device buffers and events of the pipelined process_stream, pooled
// per device across calls and plans (pinning is slow: ~10x a memcpy, and the
// drop-in creates a plan per process_stream call).
struct PsBuffers {
    static constexpr int KH = 3, KD = 2, KO = 3;
    // byte capacity of each buffer set: the reuse check compares bytes, never
    // row counts (a pooled set may have been sized for another row size)
    uint64_t hin_cap = 0, din_cap = 0, out_cap = 0;
    void* h_in[KH] = {};
    void* h_out[KO] = {};
    void* d_in[KD] = {};
    void* d_out[KO] = {};
    cudaEvent_t ev_hin[KH] = {}, ev_din[KD] = {}, ev_comp[KD] = {}, ev_d2h[KO] = {};
    void release() {
        for (auto& b : h_in)
            if (b)
                cudaFreeHost(b), b = nullptr;
        for (auto& b : h_out)
            if (b)
                cudaFreeHost(b), b = nullptr;
        for (auto& b : d_in)
            if (b)
                cudaFree(b), b = nullptr;
        for (auto& b : d_out)
            if (b)
                cudaFree(b), b = nullptr;
        for (auto& e : ev_hin)
            if (e)
                cudaEventDestroy(e), e = nullptr;
        for (auto& e : ev_din)
            if (e)
                cudaEventDestroy(e), e = nullptr;
        for (auto& e : ev_comp)
            if (e)
                cudaEventDestroy(e), e = nullptr;
        for (auto& e : ev_d2h)
            if (e)
                cudaEventDestroy(e), e = nullptr;
        hin_cap = din_cap = out_cap = 0;
    }
    // (re)allocate for blocks of io bytes (+ one spectrum of carry) of
    // row_bytes-byte spectra behind T-1 history rows
    bool ensure(uint64_t io_, uint64_t row_bytes, uint64_t T) {
        const uint64_t rows = io_ / row_bytes + 1;
        const uint64_t need_hin = io_ + row_bytes;
        const uint64_t need_din = (T - 1 + rows) * row_bytes;
        const uint64_t need_out = rows * row_bytes;
        if (hin_cap >= need_hin && din_cap >= need_din && out_cap >= need_out)
            return true;
        release();
        bool ok = true;
        for (int i = 0; i < KH && ok; ++i)
            ok = cudaMallocHost(&h_in[i], need_hin) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ev_hin[i], cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; i < KO && ok; ++i)
            ok = cudaMallocHost(&h_out[i], need_out) == cudaSuccess &&
                 cudaMalloc(&d_out[i], need_out) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ev_d2h[i], cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; i < KD && ok; ++i)
            ok = cudaMalloc(&d_in[i], need_din) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ev_din[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&ev_comp[i], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {
            release();
            cudaGetLastError();
            return false;
        }
        hin_cap = need_hin;
        din_cap = need_din;
        out_cap = need_out;
        return true;
    }
};

// ================================================================== plans
struct ppfg_plan_s {
    int device = 0;
    uint64_t C = 0, T = 0;
    uint32_t flags = 0;
    int L = -1; // log2 C when C is a power of two
    int num_sms = 148;
    float* d_taps = nullptr;     // [T][C] f32
    float2* d_tw = nullptr;      // FftPlan twiddles (wr, wi), C-1 entries
    float4* d_tw4 = nullptr;     // the same, pre-expanded (wr, wi, -wi, wr)
    double2* d_roots = nullptr;  // dft_naive roots, C entries (non-pow2)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    const FusedEntry* fused = nullptr;
    const FusedEntry* fused_power = nullptr; // detection-only configuration, if any
    std::string fused_name; // the fused kernel's configuration, as ncu prints it
    // K7 (l2x.cuh): the exchange ring + its counters (grow-only) and an event
    // ordering launches that share them
    const L2xEntry* l2x = nullptr;
    void* d_ring = nullptr;
    size_t ring_bytes = 0;
    cudaEvent_t ev_ring = nullptr;
    // host-mode pipeline buffers (grow-only)
    void* d_in[2] = {nullptr, nullptr};
    void* d_out[2] = {nullptr, nullptr};
    size_t d_in_bytes = 0, d_out_bytes = 0;
    void* h_in[2] = {nullptr, nullptr}; // pinned staging for pageable callers
    void* h_out[2] = {nullptr, nullptr};
    size_t h_in_bytes = 0, h_out_bytes = 0;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
    // detection: per-CTA partial power sums (grow-only)
    double* d_part = nullptr;
    size_t part_bytes = 0;
    void* d_bins = nullptr; // bins of the unfused detection path
    size_t bins_bytes = 0;
};

// Process-wide pool of PsBuffers per device, kept until exit like a caching
// allocator: concurrent streams each take their own, idle ones are reused.
struct PsPool {
    std::mutex mu;
    std::map<int, std::vector<PsBuffers*>> idle;
    PsBuffers* acquire(int device) {
        std::lock_guard<std::mutex> lk(mu);
        auto& v = idle[device];
        if (v.empty())
            return new PsBuffers();
        PsBuffers* b = v.back();
        v.pop_back();
        return b;
    }
    void give_back(int device, PsBuffers* b) {
        std::lock_guard<std::mutex> lk(mu);
        idle[device].push_back(b);
    }
};
PsPool& ps_pool() {
    static PsPool* pool = new PsPool(); // never destroyed: no teardown-order issues at exit
    return *pool;
}

namespace {

// FftPlan twiddles exactly as dft.hpp:88-98: double angle -> cos/sin -> f32,
// stored as (wr, wi, -wi, wr) for the packed butterfly (common.cuh bfly2).
std::vector<float2> host_twiddles(uint64_t n) {
    std::vector<float2> tw(n > 1 ? n - 1 : 1);
    for (uint64_t len = 2; len <= n; len <<= 1) {
        const uint64_t half = len / 2;
        for (uint64_t j = 0; j < half; ++j) {
            const double angle = -2.0 * M_PI * static_cast<double>(j) / static_cast<double>(len);
            const float wr = static_cast<float>(std::cos(angle));
            const float wi = static_cast<float>(std::sin(angle));
            tw[half - 1 + j] = make_float2(wr, wi);
        }
    }
    return tw;
}

// dft_naive roots (dft.hpp:47-51)
std::vector<double2> host_roots(uint64_t n) {
    std::vector<double2> r(n);
    for (uint64_t j = 0; j < n; ++j) {
        const double angle = -2.0 * M_PI * static_cast<double>(j) / static_cast<double>(n);
        r[j] = make_double2(std::cos(angle), std::sin(angle));
    }
    return r;
}

int stream_of(ppfg_plan p, void* s, cudaStream_t* out) {
    *out = s ? static_cast<cudaStream_t>(s) : p->stream;
    return PPFG_OK;
}

// ---------------------------------------------------------- launchers (device)
int encode_rows_map(CUtensorMap* map, const float2* din, uint64_t C, uint64_t S_in, int cpw, int rb);

// K1b launch: one CTA per (32-channel block, time segment); segments sized
// so the grid is a whole number of co-resident waves and the (T-1)-row halo
// each segment re-reads stays small. false if no K1b shape applies.
bool launch_fir_block(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st,
                      bool exact, double init, int* rc) {
    const uint64_t C = p->C, T = p->T;
    if ((p->flags & (PPFG_FIR_LEGACY | PPFG_K1_PREFETCH)) || C % 2 || reinterpret_cast<uintptr_t>(din) % 16)
        return false;
    const FirBlkEntry e = fir_blk_table(static_cast<int>(T), exact);
    if (!e.fn)
        return false;
    *rc = ensure_smem_attr(e.fn, e.smem, p->device);
    if (*rc != PPFG_OK)
        return true;
    const uint64_t S_out = S_in - T + 1;
    const uint64_t n_cb = cdiv(C, 32);
    // ~1024-row time segments, segment-major over the channel blocks: one
    // narrow front through the input (the halo rows come from L2); the former
    // few-waves layout with 1000+-row segments per CTA measured 1-2 % slower
    // (1 GiB FIR alone T=16 0.751 -> 0.761, T=32 0.456 -> 0.465)
    uint64_t seg = std::min<uint64_t>(std::max<uint64_t>(std::max<uint64_t>(1024, 8 * T), 4 * e.rb), S_out);
    seg = cdiv(seg, static_cast<uint64_t>(e.rb)) * e.rb; // whole steps
    const uint64_t n_seg = cdiv(S_out, seg);
    CUtensorMap map;
    *rc = encode_rows_map(&map, din, C, S_in, 32, e.rb);
    if (*rc != PPFG_OK)
        return true;
    unsigned Cu = static_cast<unsigned>(C);
    long long S_out_ll = static_cast<long long>(S_out);
    int seg_i = static_cast<int>(seg);
    void* args[] = {&map, &dout, &Cu, &S_out_ll, &p->d_taps, &seg_i, &init};
    *rc = cudaLaunchKernel(e.fn, dim3(static_cast<unsigned>(n_seg * n_cb)), dim3(e.nt), args, e.smem,
                           st) == cudaSuccess
              ? check_launch(exact ? "fir kernel (register-blocked)" : "fir kernel (register-blocked, FP32)")
              : fail(PPFG_CUDA_ERROR, "fir kernel (register-blocked): launch failed");
    return true;
}

int launch_fir(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st,
               bool reference_order) {
    const uint64_t T = p->T, C = p->C;
    const uint64_t S_out = S_in - T + 1;
    const double init = reference_order ? 0.0 : -0.0;
    long long S_in_ll = static_cast<long long>(S_in), S_out_ll = static_cast<long long>(S_out);
    unsigned Cu = static_cast<unsigned>(C);
    int rc_blk = PPFG_OK;
    if (launch_fir_block(p, din, S_in, dout, st, true, init, &rc_blk))
        return rc_blk;
    // TMA needs 16-byte-aligned rows (even C) and base address
    const bool tma_ok = !(p->flags & PPFG_K1_PREFETCH) && (C % 2 == 0) &&
                        (reinterpret_cast<uintptr_t>(din) % 16 == 0);
    const FirTmaEntry et = tma_ok ? fir_tma_table(static_cast<int>(T)) : FirTmaEntry{};
    if (et.fn) {
        const uint64_t cpw = 32 / et.k;
        const uint64_t n_cb = cdiv(C, cpw);
        // short time segments, all channel blocks of a segment in consecutive
        // tasks: the grid sweeps the input as one narrow front (each segment's
        // T-1 halo rows were just read by the previous segment: L2 hits).
        // 1 GiB, C=1024: T=8 0.903 -> 0.951 of the HBM roofline at 128 rows
        // (the previous ~440-row segments), T=4 0.913 -> 0.981 at 64 rows
        const uint64_t seg = std::min<uint64_t>(std::max<uint64_t>(64, 16 * T), S_out);
        const uint64_t n_seg = cdiv(S_out, seg);
        long long n_tasks = static_cast<long long>(n_seg * n_cb);
        int seg_i = static_cast<int>(seg);
        const unsigned blocks = static_cast<unsigned>(cdiv(static_cast<uint64_t>(n_tasks), 8));
        CUtensorMap map;
        PPFG_TRY(encode_rows_map(&map, din, C, S_in, static_cast<int>(cpw), et.rb));
        PPFG_TRY(ensure_smem_attr(et.fn, et.smem, p->device));
        void* args[] = {&map, &dout, &Cu, &S_out_ll, &p->d_taps, &seg_i, &n_tasks,
                        const_cast<double*>(&init)};
        PPFG_CUDA(cudaLaunchKernel(et.fn, dim3(blocks), dim3(256), args, et.smem, st));
        return check_launch("fir kernel (TMA)");
    }
    const FirEntry e = fir_table(static_cast<int>(T));
    if (e.fn) {
        // warp tasks = (channel block of 32/K channels) x (time segment); segments
        // long enough that the (TC-1) prefill and (K-1) pipeline drain stay small,
        // and enough tasks to keep ~4 waves of 48 warps per SM busy.
        const uint64_t cpw = 32 / e.k;
        const uint64_t n_cb = cdiv(C, cpw);
        const uint64_t target_tasks = static_cast<uint64_t>(p->num_sms) * 48 * 4;
        uint64_t seg = cdiv(S_out * n_cb, target_tasks);
        seg = std::max<uint64_t>(seg, std::min<uint64_t>(std::max<uint64_t>(32, 2 * T), S_out));
        const uint64_t n_seg = cdiv(S_out, seg);
        long long n_tasks = static_cast<long long>(n_seg * n_cb);
        int seg_i = static_cast<int>(seg);
        const unsigned blocks = static_cast<unsigned>(cdiv(static_cast<uint64_t>(n_tasks) * 32, 256));
        void* args[] = {&din, &dout, &Cu, &S_in_ll, &S_out_ll, &p->d_taps, &seg_i, &n_tasks,
                        const_cast<double*>(&init)};
        PPFG_CUDA(cudaLaunchKernel(e.fn, dim3(blocks), dim3(256), args, 0, st));
        return check_launch("fir kernel");
    }
    const uint64_t target_threads = static_cast<uint64_t>(p->num_sms) * 2048 * 2;
    uint64_t seg = std::max<uint64_t>(cdiv(S_out * C, target_threads), 1);
    const uint64_t n_work = cdiv(S_out, seg) * C;
    fir_exact_generic_kernel<<<static_cast<unsigned>(cdiv(n_work, 256)), 256, 0, st>>>(
        din, dout, Cu, static_cast<unsigned>(T), S_out_ll, p->d_taps, static_cast<int>(seg),
        static_cast<long long>(n_work), init);
    return check_launch("fir kernel (generic T)");
}

// bit-exact radix-2 for any power-of-two size via global memory (large N)
__global__ void fft_bitrev_kernel(const float2* in, float2* out, int L, long long n_rows) {
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long N = 1LL << L;
    if (g >= n_rows * N)
        return;
    const long long row = g >> L;
    const unsigned p = static_cast<unsigned>(g & (N - 1));
    out[g] = in[row * N + (__brev(p) >> (32 - L))];
}

__global__ void fft_stage_kernel(float2* data, const float2* __restrict__ tw, int L, int s,
                                 long long n_rows) {
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long half = 1LL << (s - 1);
    const long long pairs = 1LL << (L - 1);
    if (g >= n_rows * pairs)
        return;
    const long long row = g >> (L - 1);
    const long long q = g & (pairs - 1);
    const long long j = q & (half - 1);
    const long long base = (q >> (s - 1)) << s;
    float2* r = data + (row << L);
    float2 lo = r[base + j], hi = r[base + j + half];
    bfly2(lo, hi, tw_expand(tw[half - 1 + j]));
    r[base + j] = lo;
    r[base + j + half] = hi;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    return encode;
}

// Input view of the split kernel's TMA copies: 8-byte elements (c64 bytes,
// moved untouched), dims {C/R channels, R runs, S_in spectra}; a box
// {RUN, R, RB} at {rank*RUN, 0, row} is RB spectra x R runs of RUN channels.
int encode_input_map(CUtensorMap* map, const float2* din, uint64_t C, uint64_t S_in, int r, int rb,
                     int run, int box_r) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode)
        return fail(PPFG_CUDA_ERROR, "cuTensorMapEncodeTiled is not available from the driver");
    const cuuint64_t dims[3] = {C / r, static_cast<cuuint64_t>(r), S_in};
    const cuuint64_t strides[2] = {C / r * sizeof(float2), C * sizeof(float2)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(run), static_cast<cuuint32_t>(box_r),
                               static_cast<cuuint32_t>(rb)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult res = encode(map, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<float2*>(din), dims,
                                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS)
        return fail(PPFG_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(res) + ")");
    return PPFG_OK;
}

// K1t input view: 8-byte elements, dims {C channels, S_in spectra}; a box
// {cpw, rb} at {c0, row} is rb spectra of cpw consecutive channels.
int encode_rows_map(CUtensorMap* map, const float2* din, uint64_t C, uint64_t S_in, int cpw, int rb) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (!encode)
        return fail(PPFG_CUDA_ERROR, "cuTensorMapEncodeTiled is not available from the driver");
    const cuuint64_t dims[2] = {C, S_in};
    const cuuint64_t strides[1] = {C * sizeof(float2)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(cpw), static_cast<cuuint32_t>(rb)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult res = encode(map, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, const_cast<float2*>(din), dims,
                                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS)
        return fail(PPFG_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(res) + ")");
    return PPFG_OK;
}

// fn: the kernel to launch (default e->fn; e->power_fn for detection, whose
// dout is the partials buffer); *grid_out receives the CTA count
int launch_fused_entry(ppfg_plan p, const FusedEntry* e, const float* taps, uint64_t T,
                       const float2* din, uint64_t S_in, float2* dout, cudaStream_t st,
                       KernelFn fn = nullptr, uint64_t* grid_out = nullptr) {
    if (!fn)
        fn = e->fn;
    PPFG_TRY(ensure_smem_attr(fn, e->smem, p->device));
    const uint64_t S_out = S_in - T + 1;
    long long S_out_ll = static_cast<long long>(S_out);
    if (e->q > 1) {
        // one cluster of q CTAs per q SMs, all clusters co-resident (persistent)
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = e->q;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(e->nt);
        cfg.dynamicSmemBytes = e->smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(p->num_sms / e->q * e->q);
        int max_clusters = 0;
        PPFG_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg));
        if (max_clusters < 1)
            return fail(PPFG_CUDA_ERROR, "fused cluster kernel: no cluster fits an SM group");
        const uint64_t n_clusters = std::max<uint64_t>(
            1, std::min<uint64_t>(max_clusters, cdiv(S_out, e->rows_per_batch)));
        cfg.gridDim = dim3(static_cast<unsigned>(n_clusters * e->q));
        if (grid_out)
            *grid_out = n_clusters * e->q;
        long long rows_per_cluster = static_cast<long long>(cdiv(S_out, n_clusters));
        if (e->map_r > 0) {
            CUtensorMap map;
            PPFG_TRY(encode_input_map(&map, din, p->C, S_in, e->map_r, e->map_rb, e->map_run, e->map_box_r));
            void* tw = e->tw4 ? static_cast<void*>(p->d_tw4) : static_cast<void*>(p->d_tw);
            void* args[] = {&map, &din, &dout, &S_out_ll, &rows_per_cluster, &taps, &tw};
            PPFG_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
            return check_launch("fused split fir+fft kernel");
        }
        void* tw = e->tw4 ? static_cast<void*>(p->d_tw4) : static_cast<void*>(p->d_tw);
        void* args[] = {&din, &dout, &S_out_ll, &rows_per_cluster, &taps, &tw};
        PPFG_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
        return check_launch("fused cluster fir+fft kernel");
    }
    const uint64_t grid =
        std::max<uint64_t>(1, std::min<uint64_t>(p->num_sms, cdiv(S_out, e->rows_per_batch)));
    long long rows_per_cta = static_cast<long long>(cdiv(S_out, grid));
    if (grid_out)
        *grid_out = grid;
    void* tw = e->tw4 ? static_cast<void*>(p->d_tw4) : static_cast<void*>(p->d_tw);
    void* args[] = {&din, &dout, &S_out_ll, &rows_per_cta, &taps, &tw};
    PPFG_CUDA(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(e->nt), args,
                               e->smem, st));
    return check_launch("fused fir+fft kernel");
}

int launch_channelize(ppfg_plan p, const float2* din, uint64_t rows, float2* dout,
                      bool fft_fallback, cudaStream_t st) {
    if (rows == 0)
        return PPFG_OK;
    const uint64_t C = p->C;
    if (C == 1) { // a 1-point DFT is the identity (both FftPlan(1) and dft_naive)
        if (din != dout)
            PPFG_CUDA(cudaMemcpyAsync(dout, din, rows * sizeof(float2), cudaMemcpyDeviceToDevice,
                                      st));
        return PPFG_OK;
    }
    if (!is_pow2(C)) {
        if (!fft_fallback)
            return fail(PPFG_UNSUPPORTED_SIZE,
                        "channelize_block: non-power-of-two channel count with fallback disabled");
        const float2* src = din;
        if (din == dout) { // dft_naive reads the whole row for every bin: not in place
            void* tmp = nullptr;
            PPFG_CUDA(cudaMallocAsync(&tmp, rows * C * sizeof(float2), st));
            PPFG_CUDA(cudaMemcpyAsync(tmp, din, rows * C * sizeof(float2),
                                      cudaMemcpyDeviceToDevice, st));
            src = static_cast<const float2*>(tmp);
        }
        const uint64_t n = rows * C;
        dft_naive_kernel<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0, st>>>(
            src, dout, static_cast<unsigned>(C), static_cast<long long>(rows), p->d_roots);
        int rc = check_launch("dft_naive kernel");
        if (src != din)
            cudaFreeAsync(const_cast<float2*>(src), st);
        return rc;
    }
    const int L = p->L;
    // K2n (C = 64..8192): non-persistent tiles of rows (in place is safe: a
    // CTA reads all its rows before it writes any, and no other CTA touches
    // them); TMA needs a 16-byte-aligned source
    if (L >= 6 && L <= 13 && reinterpret_cast<uintptr_t>(din) % 16 == 0) {
        const FftEntry e = fft_tiles_entry(L);
        PPFG_TRY(ensure_smem_attr(e.fn, e.smem, p->device));
        const uint64_t grid = cdiv(rows, static_cast<uint64_t>(e.rows_per_tile));
        long long rows_ll = static_cast<long long>(rows);
        void* args[] = {&din, &dout, &rows_ll, &p->d_tw};
        PPFG_CUDA(cudaLaunchKernel(e.fn, dim3(static_cast<unsigned>(grid)), dim3(e.nt), args, e.smem,
                                   st));
        return check_launch("fft kernel (tiles)");
    }
    if (const FftEntry* e = fft_table(L)) {
        PPFG_TRY(ensure_smem_attr(e->fn, e->smem, p->device));
        const uint64_t tiles = cdiv(rows, static_cast<uint64_t>(e->rows_per_tile));
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e->fn, e->nt, e->smem);
        per_sm = std::max(per_sm, 1);
        const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(p->num_sms) * per_sm);
        long long rows_ll = static_cast<long long>(rows);
        void* args[] = {&din, &dout, &rows_ll, &p->d_tw};
        PPFG_CUDA(cudaLaunchKernel(e->fn, dim3(static_cast<unsigned>(grid)), dim3(e->nt), args,
                                   e->smem, st));
        return check_launch("fft kernel");
    }
    // L > kFftMaxL: bit reversal then one launch per stage, in global memory
    float2* buf = dout;
    void* tmp = nullptr;
    if (din == dout) {
        PPFG_CUDA(cudaMallocAsync(&tmp, rows * C * sizeof(float2), st));
        buf = static_cast<float2*>(tmp);
    }
    const long long n = static_cast<long long>(rows * C);
    fft_bitrev_kernel<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0, st>>>(
        din, buf, L, static_cast<long long>(rows));
    PPFG_TRY(check_launch("fft bitrev"));
    for (int s = 1; s <= L; ++s) {
        fft_stage_kernel<<<static_cast<unsigned>(cdiv(n / 2, 256)), 256, 0, st>>>(
            buf, p->d_tw, L, s, static_cast<long long>(rows));
        PPFG_TRY(check_launch("fft stage"));
    }
    if (tmp) {
        PPFG_CUDA(cudaMemcpyAsync(dout, tmp, rows * C * sizeof(float2), cudaMemcpyDeviceToDevice,
                                  st));
        cudaFreeAsync(tmp, st);
    }
    return PPFG_OK;
}

int launch_fused(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st) {
    return launch_fused_entry(p, p->fused, p->d_taps, p->T, din, S_in, dout, st);
}

// Unfused: K1 writes the filtered spectra into the output buffer, K2
// transforms them in place. (Chunking this into L2-resident pieces was
// measured slower: per-chunk waves and launches cost more than the DRAM
// round trip saves.)
// K1f: FP32 FIR (PPFG_FAST only), TMA-staged; false if no kernel applies
bool launch_fir_fast(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st,
                     int* rc) {
    const uint64_t C = p->C, T = p->T;
    if (launch_fir_block(p, din, S_in, dout, st, false, -0.0, rc))
        return true;
    const FirTmaEntry et = fir_fast_table(static_cast<int>(T));
    if (!et.fn || C % 2 || reinterpret_cast<uintptr_t>(din) % 16)
        return false;
    const uint64_t S_out = S_in - T + 1;
    const uint64_t cpw = 32 / et.k;
    const uint64_t n_cb = cdiv(C, cpw);
    // short segments, one narrow front (as launch_fir's K1t)
    const uint64_t seg = std::min<uint64_t>(std::max<uint64_t>(64, 16 * T), S_out);
    long long n_tasks = static_cast<long long>(cdiv(S_out, seg) * n_cb);
    int seg_i = static_cast<int>(seg);
    unsigned Cu = static_cast<unsigned>(C);
    long long S_out_ll = static_cast<long long>(S_out);
    const unsigned blocks = static_cast<unsigned>(cdiv(static_cast<uint64_t>(n_tasks), 8));
    CUtensorMap map;
    *rc = encode_rows_map(&map, din, C, S_in, static_cast<int>(cpw), et.rb);
    if (*rc == PPFG_OK)
        *rc = ensure_smem_attr(et.fn, et.smem, p->device);
    if (*rc != PPFG_OK)
        return true;
    void* args[] = {&map, &dout, &Cu, &S_out_ll, &p->d_taps, &seg_i, &n_tasks};
    *rc = cudaLaunchKernel(et.fn, dim3(blocks), dim3(256), args, et.smem, st) == cudaSuccess
              ? check_launch("fir kernel (FP32, FAST)")
              : fail(PPFG_CUDA_ERROR, "fir kernel (FP32, FAST): launch failed");
    return true;
}

// TMA (bulk and tensor copies) reads need a 16-byte-aligned source; a caller's
// buffer that is only 8-byte aligned (e.g. a view starting at an odd sample)
// takes the plain-load kernels instead
bool aligned16(const void* ptr) { return reinterpret_cast<uintptr_t>(ptr) % 16 == 0; }

bool tiny_exact(ppfg_plan p) { return !(p->flags & PPFG_FAST) || p->L == 0; }

// K6: tiny power-of-two C (1..32), one warp-level kernel (tiny.cuh). Lane
// groups of C lanes take contiguous time segments (a multiple of T spectra,
// enough segments for ~4 waves of 48 warps per SM).
bool launch_tiny(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st, int* rc) {
    if (p->L < 0 || p->L > 5 || (p->flags & PPFG_UNFUSED))
        return false;
    // C = 1 is the FIR alone, whose north-star bar (1e-6) an FP32 chain misses
    // at T >= 16: it always takes the FP64 (bit-exact) variant
    const KernelFn fn = tiny_table(p->L, static_cast<int>(p->T), tiny_exact(p));
    if (!fn)
        return false;
    const uint64_t T = p->T, S_out = S_in - T + 1;
    if (p->L == 0) { // fir_c1_kernel: one warp per segment of whole 32-spectrum steps
        const uint64_t target = static_cast<uint64_t>(p->num_sms) * 48 * 4;
        uint64_t seg = std::max<uint64_t>(cdiv(S_out, target), 32);
        seg = cdiv(seg, 32) * 32;
        long long n_tasks = static_cast<long long>(cdiv(S_out, seg));
        long long S_in_ll = static_cast<long long>(S_in), S_out_ll = static_cast<long long>(S_out);
        int seg_i = static_cast<int>(seg);
        void* args[] = {&din, &dout, &S_in_ll, &S_out_ll, &p->d_taps, &seg_i, &n_tasks};
        *rc = cudaLaunchKernel(fn, dim3(static_cast<unsigned>(cdiv(static_cast<uint64_t>(n_tasks) * 32, 256))),
                               dim3(256), args, 0, st) == cudaSuccess
                  ? check_launch("fir kernel (C = 1)")
                  : fail(PPFG_CUDA_ERROR, "fir kernel (C = 1): launch failed");
        return true;
    }
    // tiny.cuh: the step loop's unroll max(T, PF) (segments are whole unrolls)
    const bool pf16 = T == 16 || (T == 8 && (tiny_exact(p) || p->L <= 3));
    const uint64_t unroll = std::max<uint64_t>(T, pf16 ? 16 : 8);
    const uint64_t groups_per_warp = 32 >> p->L;
    const uint64_t target = static_cast<uint64_t>(p->num_sms) * 48 * 4 * groups_per_warp;
    uint64_t seg = std::max<uint64_t>(cdiv(S_out, target), std::min<uint64_t>(S_out, 4 * T));
    seg = cdiv(seg, unroll) * unroll;
    const long long n_tasks = static_cast<long long>(cdiv(S_out, seg));
    const uint64_t warps = cdiv(static_cast<uint64_t>(n_tasks), groups_per_warp);
    long long S_in_ll = static_cast<long long>(S_in), S_out_ll = static_cast<long long>(S_out);
    int seg_i = static_cast<int>(seg);
    long long nt = n_tasks;
    void* args[] = {&din, &dout, &S_in_ll, &S_out_ll, &p->d_taps, &p->d_tw, &seg_i, &nt};
    *rc = cudaLaunchKernel(fn, dim3(static_cast<unsigned>(cdiv(warps * 32, 256))), dim3(256), args, 0, st) ==
                  cudaSuccess
              ? check_launch("tiny fused fir+fft kernel")
              : fail(PPFG_CUDA_ERROR, "tiny fused fir+fft kernel: launch failed");
    return true;
}

// K7: one persistent CTA per SM; the exchange ring and its counters live in
// the plan (counters zeroed per launch; launches sharing them are ordered)
int launch_l2x(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st) {
    const L2xEntry* e = p->l2x;
    // a CTA's consecutive work items lie grid / (C/32) chunks apart; the
    // deferred publication (l2x.cuh) needs that well inside the ring
    if (static_cast<uint64_t>(p->num_sms) / (p->C / 32) + 2 > static_cast<uint64_t>(e->nsr))
        return fail(PPFG_CONFIG_ERROR, "fused fir+fft (L2 exchange): ring too small for this grid");
    // counters [2 * nsr], the trace flag, then (at +256 B) the debug timeline
    const char* trace_path = std::getenv("PPFG_L2X_TRACE");
    constexpr size_t kTraceBytes = sizeof(unsigned long long) * 2 * 8 * 256;
    const size_t ctr_bytes = 256 + (trace_path ? kTraceBytes : 0);
    if (p->ring_bytes < e->ring_bytes + ctr_bytes) {
        if (p->d_ring) {
            PPFG_CUDA(cudaStreamSynchronize(st));
            cudaFree(p->d_ring);
            p->d_ring = nullptr;
            p->ring_bytes = 0;
        }
        PPFG_CUDA(cudaMalloc(&p->d_ring, e->ring_bytes + ctr_bytes));
        p->ring_bytes = e->ring_bytes + ctr_bytes;
    }
    if (!p->ev_ring)
        PPFG_CUDA(cudaEventCreateWithFlags(&p->ev_ring, cudaEventDisableTiming));
    else
        PPFG_CUDA(cudaStreamWaitEvent(st, p->ev_ring, 0)); // a previous launch on another stream
    unsigned* ctr = reinterpret_cast<unsigned*>(static_cast<char*>(p->d_ring) + e->ring_bytes);
    PPFG_CUDA(cudaMemsetAsync(ctr, 0, ctr_bytes, st));
    if (trace_path) {
        static const unsigned one = 1;
        PPFG_CUDA(cudaMemcpyAsync(ctr + 2 * e->nsr, &one, sizeof(one), cudaMemcpyHostToDevice, st));
    }
    PPFG_TRY(ensure_smem_attr(e->fn, e->smem, p->device));
    CUtensorMap map;
    PPFG_TRY(encode_rows_map(&map, din, p->C, S_in, 32, e->rb));
    long long S_out = static_cast<long long>(S_in - p->T + 1);
    float2* ring = static_cast<float2*>(p->d_ring);
    void* args[] = {&map, &dout, &ring, &ctr, &S_out, &p->d_taps, &p->d_tw};
    PPFG_CUDA(cudaLaunchKernel(e->fn, dim3(static_cast<unsigned>(p->num_sms)), dim3(e->nt), args, e->smem, st));
    PPFG_TRY(check_launch("fused fir+fft kernel (L2 exchange)"));
    PPFG_CUDA(cudaEventRecord(p->ev_ring, st));
    if (trace_path) { // debug: dump CTA 0's timeline (u64 [2][8][256], ns)
        std::vector<unsigned long long> tr(2 * 8 * 256);
        PPFG_CUDA(cudaMemcpyAsync(tr.data(), reinterpret_cast<char*>(ctr) + 256, kTraceBytes,
                                  cudaMemcpyDeviceToHost, st));
        PPFG_CUDA(cudaStreamSynchronize(st));
        if (FILE* f = std::fopen(trace_path, "wb")) {
            std::fwrite(tr.data(), 1, kTraceBytes, f);
            std::fclose(f);
        }
    }
    return PPFG_OK;
}

int launch_fir_fft(ppfg_plan p, const float2* din, uint64_t S_in, float2* dout, cudaStream_t st) {
    if (p->l2x && !(p->flags & PPFG_UNFUSED) && aligned16(din))
        return launch_l2x(p, din, S_in, dout, st);
    if (p->fused && !(p->flags & PPFG_UNFUSED) && aligned16(din))
        return launch_fused(p, din, S_in, dout, st);
    int rc_tiny = PPFG_OK;
    if (launch_tiny(p, din, S_in, dout, st, &rc_tiny))
        return rc_tiny;
    int rc = PPFG_OK;
    if ((p->flags & PPFG_FAST) && launch_fir_fast(p, din, S_in, dout, st, &rc)) {
        PPFG_TRY(rc);
        return launch_channelize(p, dout, S_in - p->T + 1, dout, true, st);
    }
    PPFG_TRY(launch_fir(p, din, S_in, dout, st, false));
    return launch_channelize(p, dout, S_in - p->T + 1, dout, true, st);
}

// -------------------------------------------------------------- detection
// Per-channel mean power of channelized spectra, cmd_inspect (cli.hpp:307-317):
// mean[c] = sum_s ((double)re^2 + (double)im^2) / n. Partial sums per CTA in
// spectrum order, then a fixed-order sum over CTAs: deterministic; it differs
// from the reference's single running sum only by summation order (relative
// ~1e-16 per term).
int ensure_parts(ppfg_plan p, size_t bytes) {
    if (p->part_bytes >= bytes)
        return PPFG_OK;
    cudaFree(p->d_part);
    p->d_part = nullptr;
    p->part_bytes = 0;
    PPFG_CUDA(cudaMalloc(&p->d_part, bytes));
    p->part_bytes = bytes;
    return PPFG_OK;
}

int launch_power_reduce(ppfg_plan p, int n_parts, uint64_t n, double* dmean, cudaStream_t st) {
    const int C = static_cast<int>(p->C);
    power_reduce_kernel<<<static_cast<unsigned>(cdiv(p->C, 256)), 256, 0, st>>>(
        p->d_part, n_parts, C, static_cast<double>(n), dmean);
    return check_launch("power reduce kernel");
}

int launch_mean_power(ppfg_plan p, const float2* bins, uint64_t n, double* dmean, cudaStream_t st) {
    const uint64_t grid = std::max<uint64_t>(
        1, std::min<uint64_t>(static_cast<uint64_t>(p->num_sms) * 8, cdiv(n, 16)));
    const long long rows = static_cast<long long>(cdiv(std::max<uint64_t>(n, 1), grid));
    const int parts = static_cast<int>(cdiv(std::max<uint64_t>(n, 1), static_cast<uint64_t>(rows)));
    PPFG_TRY(ensure_parts(p, static_cast<size_t>(parts) * p->C * sizeof(double)));
    power_partial_kernel<<<static_cast<unsigned>(parts), 256, 0, st>>>(
        bins, static_cast<long long>(n), static_cast<int>(p->C), rows, p->d_part);
    PPFG_TRY(check_launch("power partial kernel"));
    return launch_power_reduce(p, parts, n, dmean, st);
}

// FIR -> FFT -> mean power. With a detection variant of the fused kernel the
// bins never reach HBM (the pass is read-only: 8*C*S_in bytes); otherwise the
// bins go through a temporary buffer.
int launch_fir_fft_mean_power(ppfg_plan p, const float2* din, uint64_t S_in, double* dmean,
                              cudaStream_t st) {
    const uint64_t S_out = S_in - p->T + 1;
    const FusedEntry* e = p->fused_power && p->fused ? p->fused_power : p->fused;
    if (e && e->power_fn && !(p->flags & PPFG_UNFUSED) && aligned16(din)) {
        // partials: at most one CTA per SM, power_rows rows of C doubles each
        PPFG_TRY(ensure_parts(p, static_cast<size_t>(p->num_sms) * e->power_rows * p->C * sizeof(double)));
        uint64_t grid = 0;
        PPFG_TRY(launch_fused_entry(p, e, p->d_taps, p->T, din, S_in,
                                    reinterpret_cast<float2*>(p->d_part), st, e->power_fn, &grid));
        return launch_power_reduce(p, static_cast<int>(grid) * e->power_rows, S_out, dmean, st);
    }
    // bins through a plan-owned (grow-only) buffer; the stream orders reuse
    const size_t bytes = S_out * p->C * sizeof(float2);
    if (p->bins_bytes < bytes) {
        cudaFree(p->d_bins);
        p->d_bins = nullptr;
        p->bins_bytes = 0;
        PPFG_CUDA(cudaMalloc(&p->d_bins, bytes));
        p->bins_bytes = bytes;
    }
    float2* bins = static_cast<float2*>(p->d_bins);
    PPFG_TRY(launch_fir_fft(p, din, S_in, bins, st));
    return launch_mean_power(p, bins, S_out, dmean, st);
}

// host buffers: stage the input in device memory, run, read the C means back
int run_mean_power(ppfg_plan p, bool fused, const void* in, uint64_t n_rows, double* mean, int mem,
                   void* s) {
    DeviceGuard dg(p->device);
    cudaStream_t st;
    stream_of(p, s, &st);
    if (mem == PPFG_MEM_DEVICE)
        return fused ? launch_fir_fft_mean_power(p, static_cast<const float2*>(in), n_rows, mean, st)
                     : launch_mean_power(p, static_cast<const float2*>(in), n_rows, mean, st);
    if (mem != PPFG_MEM_HOST)
        return fail(PPFG_CONFIG_ERROR, "ppfg: unknown memory kind");
    const size_t in_bytes = n_rows * p->C * sizeof(float2);
    void* din = nullptr;
    double* dmean = nullptr;
    PPFG_CUDA(cudaMallocAsync(&din, std::max<size_t>(in_bytes, 1), st));
    int rc = cudaMallocAsync(reinterpret_cast<void**>(&dmean), p->C * sizeof(double), st) == cudaSuccess
                 ? PPFG_OK
                 : fail(PPFG_CUDA_ERROR, "mean power: allocation failed");
    if (rc == PPFG_OK && in_bytes)
        rc = cudaMemcpyAsync(din, in, in_bytes, cudaMemcpyHostToDevice, st) == cudaSuccess
                 ? PPFG_OK
                 : fail(PPFG_CUDA_ERROR, "mean power: H2D copy failed");
    if (rc == PPFG_OK)
        rc = fused ? launch_fir_fft_mean_power(p, static_cast<const float2*>(din), n_rows, dmean, st)
                   : launch_mean_power(p, static_cast<const float2*>(din), n_rows, dmean, st);
    if (rc == PPFG_OK)
        rc = cudaMemcpyAsync(mean, dmean, p->C * sizeof(double), cudaMemcpyDeviceToHost, st) ==
                     cudaSuccess
                 ? PPFG_OK
                 : fail(PPFG_CUDA_ERROR, "mean power: D2H copy failed");
    cudaFreeAsync(din, st);
    cudaFreeAsync(dmean, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == PPFG_OK)
        rc = fail(PPFG_CUDA_ERROR, "mean power: stream error");
    return rc;
}

// ------------------------------------------------------ host copy pool
// Pageable callers (the reference API hands over std::vectors) pay a host
// copy into / out of pinned staging per call; one core copies ~8-10 GB/s,
// below PCIe, so large copies are split over a small process-wide pool of
// worker threads (they also take the first-touch page faults of freshly
// allocated output vectors in parallel). Each piece is copied by
// ppfg::copy_piece (hostcopy.cpp: streaming stores for large pieces).

class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool(); // never destroyed: no teardown-order issues
        return *p;
    }
    void copy(void* dst, const void* src, size_t bytes) {
        // 1 MiB pieces: an 8 MiB staging chunk goes to all 8 threads
        constexpr size_t kPiece = size_t(1) << 20;
        if (bytes < 2 * kPiece || n_workers_ == 0) {
            ppfg::copy_piece(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one(job_mu_); // one parallel copy at a time
        const size_t parts = std::min<size_t>(n_workers_ + 1, bytes / kPiece);
        job_dst_ = static_cast<char*>(dst);
        job_src_ = static_cast<const char*>(src);
        job_bytes_ = bytes;
        job_per_ = ((bytes + parts - 1) / parts + 63) & ~size_t(63); // parts * per >= bytes
        job_parts_ = parts;
        done_.store(0, std::memory_order_relaxed);
        const uint64_t g = ++gen_;
        // publish: the job fields happen-before any claim of generation g
        next_.store(g << 32, std::memory_order_release);
        {
            std::lock_guard<std::mutex> lk(mu_);
            wake_ = g;
        }
        cv_.notify_all();
        work(g);
        std::unique_lock<std::mutex> lk(mu_);
        cv_done_.wait(lk, [&] { return done_.load(std::memory_order_acquire) == parts; });
    }

private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        n_workers_ = hw > 2 ? std::min(hw - 1, 7u) : 0u;
        for (unsigned i = 0; i < n_workers_; ++i)
            std::thread([this] { loop(); }).detach();
    }
    // claim parts of generation g (index in the low 32 bits of next_) until
    // none is left; a part claimed keeps the job (and its fields) alive
    void work(uint64_t g) {
        size_t finished = 0;
        for (;;) {
            uint64_t v = next_.load(std::memory_order_acquire);
            if ((v >> 32) != g || (v & 0xffffffffu) >= job_parts_)
                break;
            if (!next_.compare_exchange_weak(v, v + 1, std::memory_order_acq_rel))
                continue;
            const size_t o = (v & 0xffffffffu) * job_per_;
            if (o < job_bytes_)
                ppfg::copy_piece(job_dst_ + o, job_src_ + o, std::min(job_per_, job_bytes_ - o));
            ++finished;
        }
        if (finished && done_.fetch_add(finished, std::memory_order_acq_rel) + finished == job_parts_) {
            std::lock_guard<std::mutex> lk(mu_);
            cv_done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return wake_ != seen; });
                seen = wake_;
            }
            work(seen);
        }
    }
    unsigned n_workers_ = 0;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, cv_done_;
    uint64_t gen_ = 0, wake_ = 0;
    char* job_dst_ = nullptr;
    const char* job_src_ = nullptr;
    size_t job_bytes_ = 0, job_per_ = 0, job_parts_ = 0;
    std::atomic<uint64_t> next_{0};
    std::atomic<size_t> done_{0};
};

void host_copy(void* dst, const void* src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

// ------------------------------------------------------ host-mode pipeline
bool is_pinned(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

int grow_device(void** bufs, size_t* have, size_t need) {
    if (*have >= need)
        return PPFG_OK;
    for (int i = 0; i < 2; ++i) {
        if (bufs[i])
            cudaFree(bufs[i]);
        bufs[i] = nullptr;
    }
    for (int i = 0; i < 2; ++i)
        PPFG_CUDA(cudaMalloc(&bufs[i], need));
    *have = need;
    return PPFG_OK;
}

int grow_pinned(void** bufs, size_t* have, size_t need) {
    if (*have >= need)
        return PPFG_OK;
    for (int i = 0; i < 2; ++i) {
        if (bufs[i])
            cudaFreeHost(bufs[i]);
        bufs[i] = nullptr;
    }
    for (int i = 0; i < 2; ++i)
        PPFG_CUDA(cudaHostAlloc(&bufs[i], need, cudaHostAllocDefault));
    *have = need;
    return PPFG_OK;
}

enum class Op { Fir, FirRef, Channelize, ChannelizeNoFallback, FirFft };

int launch_op(ppfg_plan p, Op op, const float2* din, uint64_t n_in_rows, float2* dout,
              cudaStream_t st) {
    switch (op) {
    case Op::Fir:
        return launch_fir(p, din, n_in_rows, dout, st, false);
    case Op::FirRef:
        return launch_fir(p, din, n_in_rows, dout, st, true);
    case Op::Channelize:
        return launch_channelize(p, din, n_in_rows, dout, true, st);
    case Op::ChannelizeNoFallback:
        return launch_channelize(p, din, n_in_rows, dout, false, st);
    case Op::FirFft:
        return launch_fir_fft(p, din, n_in_rows, dout, st);
    }
    return PPFG_CONFIG_ERROR;
}

constexpr size_t kChunkBytes = size_t(64) << 20;
constexpr size_t kPageableChunkBytes = size_t(8) << 20;

// Host buffers -> chunked, double-buffered H2D | kernel | D2H on three streams.
// `halo` input rows overlap between chunks (T-1 for the FIR, 0 for the FFT);
// output row r depends on input rows r .. r+halo.
int run_host(ppfg_plan p, Op op, const void* hin, uint64_t n_in_rows, void* hout, uint64_t halo) {
    const uint64_t row_bytes = p->C * sizeof(float2);
    const uint64_t n_out_rows = n_in_rows - halo;
    if (n_out_rows == 0)
        return PPFG_OK;
    const bool pin_in = is_pinned(hin), pin_out = is_pinned(hout);
    // pageable buffers: smaller chunks, so the host staging copy of chunk i+1
    // overlaps the PCIe transfers and the kernel of chunk i
    const uint64_t chunk_bytes = pin_in && pin_out ? kChunkBytes : kPageableChunkBytes;
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(n_out_rows,
                                                                   chunk_bytes / row_bytes));
    PPFG_TRY(grow_device(p->d_in, &p->d_in_bytes, (chunk + halo) * row_bytes));
    PPFG_TRY(grow_device(p->d_out, &p->d_out_bytes, chunk * row_bytes));
    if (!pin_in)
        PPFG_TRY(grow_pinned(p->h_in, &p->h_in_bytes, (chunk + halo) * row_bytes));
    if (!pin_out)
        PPFG_TRY(grow_pinned(p->h_out, &p->h_out_bytes, chunk * row_bytes));
    const uint64_t n_chunks = cdiv(n_out_rows, chunk);
    const char* src = static_cast<const char*>(hin);
    char* dst = static_cast<char*>(hout);
    // pending host copy-out of chunk i-2 (pageable outputs)
    auto drain = [&](uint64_t i) -> int {
        const int b = static_cast<int>(i & 1);
        const uint64_t o = i * chunk, n = std::min(chunk, n_out_rows - o);
        PPFG_CUDA(cudaEventSynchronize(p->ev_d2h[b]));
        if (!pin_out)
            host_copy(dst + o * row_bytes, p->h_out[b], n * row_bytes);
        return PPFG_OK;
    };
    for (uint64_t i = 0; i < n_chunks; ++i) {
        const int b = static_cast<int>(i & 1);
        const uint64_t o = i * chunk, n = std::min(chunk, n_out_rows - o);
        const uint64_t in_bytes = (n + halo) * row_bytes, out_bytes = n * row_bytes;
        // pageable outputs: copy chunk i-2 out of its staging buffer before
        // reusing it (pinned outputs need no host sync: every reuse below is
        // ordered on the device by events, so H2D, kernels and D2H overlap)
        if (i >= 2 && !pin_out)
            PPFG_TRY(drain(i - 2));
        // input: d_in[b] is free once chunk i-2's kernel has run
        if (i >= 2)
            PPFG_CUDA(cudaStreamWaitEvent(p->s_h2d, p->ev_comp[b], 0));
        const void* h2d_src = src + o * row_bytes;
        if (!pin_in) {
            PPFG_CUDA(cudaEventSynchronize(p->ev_h2d[b])); // staging buffer reusable
            host_copy(p->h_in[b], src + o * row_bytes, in_bytes);
            h2d_src = p->h_in[b];
        }
        PPFG_CUDA(cudaMemcpyAsync(p->d_in[b], h2d_src, in_bytes, cudaMemcpyHostToDevice,
                                  p->s_h2d));
        PPFG_CUDA(cudaEventRecord(p->ev_h2d[b], p->s_h2d));
        // compute: after its input landed and chunk i-2's output left d_out[b]
        PPFG_CUDA(cudaStreamWaitEvent(p->stream, p->ev_h2d[b], 0));
        if (i >= 2)
            PPFG_CUDA(cudaStreamWaitEvent(p->stream, p->ev_d2h[b], 0));
        PPFG_TRY(launch_op(p, op, static_cast<const float2*>(p->d_in[b]), n + halo,
                           static_cast<float2*>(p->d_out[b]), p->stream));
        PPFG_CUDA(cudaEventRecord(p->ev_comp[b], p->stream));
        // output
        PPFG_CUDA(cudaStreamWaitEvent(p->s_d2h, p->ev_comp[b], 0));
        PPFG_CUDA(cudaMemcpyAsync(pin_out ? static_cast<void*>(dst + o * row_bytes) : p->h_out[b],
                                  p->d_out[b], out_bytes, cudaMemcpyDeviceToHost, p->s_d2h));
        PPFG_CUDA(cudaEventRecord(p->ev_d2h[b], p->s_d2h));
    }
    if (!pin_out)
        for (uint64_t i = n_chunks >= 2 ? n_chunks - 2 : 0; i < n_chunks; ++i)
            PPFG_TRY(drain(i));
    PPFG_CUDA(cudaStreamSynchronize(p->s_d2h));
    PPFG_CUDA(cudaStreamSynchronize(p->stream));
    return PPFG_OK;
}

int check_plan(ppfg_plan p) {
    if (!p)
        return fail(PPFG_CONFIG_ERROR, "ppfg: null plan");
    return PPFG_OK;
}

// fir.hpp:56-65 preconditions on an input of n_spectra_in spectra
int check_fir_input(ppfg_plan p, const void* in, uint64_t n_spectra_in, const void* out) {
    PPFG_TRY(check_plan(p));
    if (p->T == 0)
        return fail(PPFG_CONFIG_ERROR, "fir: malformed coefficient set");
    if (n_spectra_in == 0)
        return fail(PPFG_CONFIG_ERROR,
                    "SampleBlock: sample count must be a positive multiple of n_channels");
    if (n_spectra_in < p->T)
        return fail(PPFG_INSUFFICIENT_HISTORY, "fir: need at least n_taps input spectra");
    if (!in || !out)
        return fail(PPFG_CONFIG_ERROR, "fir: null buffer");
    return PPFG_OK;
}

int run(ppfg_plan p, Op op, const void* in, uint64_t n_in_rows, void* out, int mem, void* s,
        uint64_t halo) {
    DeviceGuard dg(p->device);
    if (mem == PPFG_MEM_DEVICE) {
        cudaStream_t st;
        stream_of(p, s, &st);
        return launch_op(p, op, static_cast<const float2*>(in), n_in_rows, static_cast<float2*>(out),
                         st);
    }
    if (mem != PPFG_MEM_HOST)
        return fail(PPFG_CONFIG_ERROR, "ppfg: unknown memory kind");
    return run_host(p, op, in, n_in_rows, out, halo);
}

// ------------------------------------------------------------ synth tables
struct ToneCache {
    std::mutex mu;
    std::map<std::pair<int, uint64_t>, float2*> dev;
};
ToneCache& tone_cache() {
    static ToneCache c;
    return c;
}

std::vector<float2> host_tone(uint64_t C) {
    const uint64_t M = 10 * C;
    std::vector<float2> t(M);
    for (uint64_t k = 0; k < M; ++k) {
        const double a = 2.0 * M_PI * static_cast<double>(k) / static_cast<double>(M);
        t[k] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
    return t;
}

uint64_t tone_f10(uint64_t C) { return (10 * C) / 8 + 3; }

// "fused_fir_fft_kernel<FusedCfg<10, 8, 2, 0, ...>>" from the entry maker's
// __PRETTY_FUNCTION__ ("... [with Cfg = ppfg::FusedCfg<10, 8, 2, false, ...>]"),
// spelled the way ncu prints the template arguments (bools as 0/1)
std::string kernel_name_of(const FusedEntry& e) {
    std::string sig = e.sig ? e.sig : "";
    const size_t at = sig.find("Cfg = ");
    std::string cfg = at == std::string::npos ? sig : sig.substr(at + 6);
    if (!cfg.empty() && cfg.back() == ']')
        cfg.pop_back();
    for (const char* ns : {"ppfg::"})
        for (size_t k; (k = cfg.find(ns)) != std::string::npos;)
            cfg.erase(k, std::strlen(ns));
    for (auto [from, to] : {std::pair<const char*, const char*>{"false", "0"}, {"true", "1"}})
        for (size_t k; (k = cfg.find(from)) != std::string::npos;)
            cfg.replace(k, std::strlen(from), to);
    return std::string(e.q > 1 ? "fused_split_kernel<" : "fused_fir_fft_kernel<") + cfg + ">";
}

// Process-wide cache of idle plans for the library's own one-shot entry
// points (ppfg_multi_fir_fft's per-device shards, the single-row fft /
// dft_naive helpers): keyed by (device, C, T, flags, coefficient values);
// a plan is leased to one call at a time and keeps its pinned staging and
// device buffers between calls. At most kMaxIdle idle plans are kept.
struct PlanLease {
    int device = 0;
    uint64_t C = 0, T = 0;
    uint32_t flags = 0;
    std::vector<double> values;
    ppfg_plan plan = nullptr;
};
struct LibPlanCache {
    static constexpr size_t kMaxIdle = 16;
    std::mutex mu;
    std::list<PlanLease> idle; // most recently used first
};
LibPlanCache& lib_plan_cache() {
    static LibPlanCache* c = new LibPlanCache(); // never destroyed: no exit-order issues
    return *c;
}
int lease_plan(uint64_t C, uint64_t T, const double* values, uint32_t flags, int device, PlanLease* out) {
    out->device = device;
    out->C = C;
    out->T = T;
    out->flags = flags;
    out->values.assign(values, values + (T ? C * T : 0));
    {
        auto& c = lib_plan_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.idle.begin(); it != c.idle.end(); ++it) {
            if (it->device == device && it->C == C && it->T == T && it->flags == flags &&
                it->values == out->values) {
                out->plan = it->plan;
                c.idle.erase(it);
                return PPFG_OK;
            }
        }
    }
    return ppfg_plan_create(&out->plan, C, T, T ? out->values.data() : nullptr, flags, device);
}
void return_plan(PlanLease&& l) {
    if (!l.plan)
        return;
    auto& c = lib_plan_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.idle.push_front(std::move(l));
    while (c.idle.size() > LibPlanCache::kMaxIdle) {
        ppfg_plan_destroy(c.idle.back().plan);
        c.idle.pop_back();
    }
}

} // namespace

// ================================================================ C-ABI
extern "C" {

const char* ppfg_version(void) { return "ppfg 0.1 (sm_100a)"; }
const char* ppfg_last_error(void) { return g_err.c_str(); }
uint64_t ppfg_last_error_offset(void) { return g_err_offset; }
uint64_t ppfg_kernel_launches(void) { return g_launches.load(); }

uint64_t ppfg_flops_for_fir(uint64_t n_channels, uint64_t n_taps, uint64_t n_spectra_out) {
    return n_spectra_out * n_channels * n_taps * 4u; // fir.hpp:49-52
}

uint64_t ppfg_flops_for_dft(uint64_t n_channels, uint64_t n_spectra) { // dft.hpp:28-35
    if (is_pow2(n_channels))
        return n_spectra * 5u * n_channels * static_cast<uint64_t>(ilog2(n_channels));
    return n_spectra * 8u * n_channels * n_channels;
}

int ppfg_plan_create(ppfg_plan* plan, uint64_t n_channels, uint64_t n_taps,
                     const double* coeff_values, uint32_t flags, int device) {
    if (!plan)
        return fail(PPFG_CONFIG_ERROR, "ppfg_plan_create: null plan pointer");
    *plan = nullptr;
    if (n_channels == 0)
        return fail(PPFG_CONFIG_ERROR, "SampleBlock: n_channels must be >= 1");
    if (n_taps > 0 && !coeff_values)
        return fail(PPFG_CONFIG_ERROR, "fir: malformed coefficient set");
    if (n_channels > (uint64_t(1) << 24) || n_taps > 4096)
        return fail(PPFG_CONFIG_ERROR, "ppfg_plan_create: channel or tap count out of range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(PPFG_NO_DEVICE, "ppfg: no CUDA device");
    }
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess) // -1: the caller's current device
        return fail(PPFG_NO_DEVICE, "ppfg: no current device");
    if (device >= ndev)
        return fail(PPFG_NO_DEVICE, "ppfg: device index out of range");
    DeviceGuard dg(device);
    cudaDeviceProp prop{};
    PPFG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(PPFG_NO_DEVICE, std::string("ppfg: needs an sm_100 device, found ") + prop.name);
    auto* p = new ppfg_plan_s();
    p->device = device;
    p->C = n_channels;
    p->T = n_taps;
    p->flags = flags;
    p->num_sms = prop.multiProcessorCount;
    p->L = is_pow2(n_channels) ? ilog2(n_channels) : -1;
    auto cleanup = [&](int st) {
        ppfg_plan_destroy(p);
        return st;
    };
    if (n_taps > 0) { // quantize_taps (fir.hpp:69-74)
        std::vector<float> taps(n_taps * n_channels);
        for (size_t k = 0; k < taps.size(); ++k)
            taps[k] = static_cast<float>(coeff_values[k]);
        if (cudaMalloc(&p->d_taps, taps.size() * sizeof(float)) != cudaSuccess ||
            cudaMemcpy(p->d_taps, taps.data(), taps.size() * sizeof(float),
                       cudaMemcpyHostToDevice) != cudaSuccess)
            return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: tap upload failed"));
    }
    if (p->L >= 1) {
        const auto tw = host_twiddles(n_channels);
        if (cudaMalloc(&p->d_tw, tw.size() * sizeof(float2)) != cudaSuccess ||
            cudaMemcpy(p->d_tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice) !=
                cudaSuccess)
            return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: twiddle upload failed"));
        std::vector<float4> tw4(tw.size());
        for (size_t i = 0; i < tw.size(); ++i)
            tw4[i] = make_float4(tw[i].x, tw[i].y, -tw[i].y, tw[i].x);
        if (cudaMalloc(&p->d_tw4, tw4.size() * sizeof(float4)) != cudaSuccess ||
            cudaMemcpy(p->d_tw4, tw4.data(), tw4.size() * sizeof(float4), cudaMemcpyHostToDevice) !=
                cudaSuccess)
            return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: twiddle upload failed"));
    } else if (p->L < 0) {
        const auto r = host_roots(n_channels);
        if (cudaMalloc(&p->d_roots, r.size() * sizeof(double2)) != cudaSuccess ||
            cudaMemcpy(p->d_roots, r.data(), r.size() * sizeof(double2),
                       cudaMemcpyHostToDevice) != cudaSuccess)
            return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: root upload failed"));
    }
    // the table uploads above are plain cudaMemcpy calls from pageable memory,
    // which may return before their DMA has landed; the plan's kernels run on
    // non-blocking streams, so wait for the legacy stream once here
    if (cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess)
        return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: table upload failed"));
    if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: stream creation failed"));
    p->own_stream = true;
    for (int i = 0; i < 2; ++i) {
        if (cudaEventCreateWithFlags(&p->ev_h2d[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_d2h[i], cudaEventDisableTiming) != cudaSuccess)
            return cleanup(fail(PPFG_CUDA_ERROR, "ppfg_plan_create: event creation failed"));
    }
    if (n_taps > 0 && p->L >= 0) {
        const bool exact = !(flags & PPFG_FAST);
        // Cluster kernels: by default only where measured faster than
        // FIR -> HBM -> FFT; PPFG_CLUSTER forces them.
        const bool want_cluster = (flags & PPFG_CLUSTER) != 0;
        for (const auto& e : fused_table()) {
            if (e.power_only && !p->fused_power && e.L == p->L && e.T == static_cast<int>(n_taps) &&
                e.exact == exact)
                p->fused_power = &e;
        }
        for (const auto& e : fused_table()) {
            if (!e.power_only && e.L == p->L && e.T == static_cast<int>(n_taps) && e.exact == exact &&
                (e.q == 1 || want_cluster || e.preferred)) {
                p->fused = &e;
                p->fused_name = kernel_name_of(e);
                break;
            }
        }
        for (const auto& e : l2x_entries()) {
            if (e.L == p->L && e.T == static_cast<int>(n_taps) && e.exact == exact &&
                (e.preferred || (flags & PPFG_L2X))) {
                p->l2x = &e;
                FusedEntry tmp{};
                tmp.sig = e.sig;
                p->fused_name = "fused_l2x_kernel<" + kernel_name_of(tmp).substr(std::strlen("fused_fir_fft_kernel<"));
                break;
            }
        }
    }
    *plan = p;
    return PPFG_OK;
}

int ppfg_plan_destroy(ppfg_plan p) {
    if (!p)
        return PPFG_OK;
    DeviceGuard dg(p->device);
    if (p->stream)
        cudaStreamSynchronize(p->stream);
    cudaFree(p->d_taps);
    cudaFree(p->d_tw);
    cudaFree(p->d_tw4);
    cudaFree(p->d_roots);
    cudaFree(p->d_part);
    cudaFree(p->d_bins);
    cudaFree(p->d_ring);
    if (p->ev_ring)
        cudaEventDestroy(p->ev_ring);

    for (int i = 0; i < 2; ++i) {
        cudaFree(p->d_in[i]);
        cudaFree(p->d_out[i]);
        if (p->h_in[i])
            cudaFreeHost(p->h_in[i]);
        if (p->h_out[i])
            cudaFreeHost(p->h_out[i]);
        if (p->ev_h2d[i])
            cudaEventDestroy(p->ev_h2d[i]);
        if (p->ev_comp[i])
            cudaEventDestroy(p->ev_comp[i]);
        if (p->ev_d2h[i])
            cudaEventDestroy(p->ev_d2h[i]);
    }
    if (p->own_stream) {
        cudaStreamDestroy(p->stream);
        cudaStreamDestroy(p->s_h2d);
        cudaStreamDestroy(p->s_d2h);
    }
    delete p;
    return PPFG_OK;
}

void* ppfg_plan_stream(ppfg_plan plan) { return plan ? plan->stream : nullptr; }

const char* ppfg_fir_fft_kernel_name(ppfg_plan p) {
    if (!p)
        return "";
    if (!(p->flags & PPFG_UNFUSED) && p->L >= 0 && p->L <= 5 && p->T > 0 &&
        tiny_table(p->L, static_cast<int>(p->T), tiny_exact(p)))
        return tiny_exact(p) ? "fused_tiny_kernel (FP64 FIR)" : "fused_tiny_kernel (FP32 FIR)";
    if (!(p->l2x || p->fused) || (p->flags & PPFG_UNFUSED))
        return "unfused (FIR kernel + FFT kernel)";
    return p->fused_name.c_str();
}

int ppfg_host_copy(void* dst, const void* src, uint64_t bytes) {
    if (bytes && (!dst || !src))
        return fail(PPFG_CONFIG_ERROR, "host_copy: null buffer");
    host_copy(dst, src, bytes);
    return PPFG_OK;
}

int ppfg_current_device(int* device) {
    if (!device)
        return fail(PPFG_CONFIG_ERROR, "current_device: null output");
    if (cudaGetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return fail(PPFG_NO_DEVICE, "ppfg: no current device");
    }
    return PPFG_OK;
}

int ppfg_device_hbm_gbs(int device, double* gbs) {
    if (!gbs)
        return fail(PPFG_CONFIG_ERROR, "device_hbm_gbs: null output");
    *gbs = 0.0;
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess)
        return fail(PPFG_NO_DEVICE, "ppfg: no current device");
    int khz = 0, bits = 0;
    if (cudaDeviceGetAttribute(&khz, cudaDevAttrMemoryClockRate, device) != cudaSuccess ||
        cudaDeviceGetAttribute(&bits, cudaDevAttrGlobalMemoryBusWidth, device) != cudaSuccess) {
        cudaGetLastError();
        return fail(PPFG_NO_DEVICE, "ppfg: cannot query the device memory system");
    }
    *gbs = 2.0 * static_cast<double>(khz) * 1e3 * static_cast<double>(bits) / 8.0 / 1e9;
    return PPFG_OK;
}

int ppfg_fir_fft_kind(ppfg_plan p) {
    if (p && !(p->flags & PPFG_UNFUSED) && p->L >= 0 && p->L <= 5 && p->T > 0 &&
        tiny_table(p->L, static_cast<int>(p->T), tiny_exact(p)))
        return tiny_exact(p) ? 6 : 5;
    if (p && p->l2x && !(p->flags & PPFG_UNFUSED))
        return p->l2x->exact ? 8 : 7;
    if (!p || !p->fused || (p->flags & PPFG_UNFUSED))
        return 0;
    return (p->fused->exact ? 2 : 1) + (p->fused->q > 1 ? 2 : 0);
}

int ppfg_fir(ppfg_plan p, const void* in, uint64_t n_spectra_in, void* out, int mem,
             void* cuda_stream) {
    PPFG_TRY(check_fir_input(p, in, n_spectra_in, out));
    if (in == out)
        return fail(PPFG_CONFIG_ERROR, "fir: input and output must not alias");
    return run(p, Op::Fir, in, n_spectra_in, out, mem, cuda_stream, p->T - 1);
}

// ppf_fir_reference's start-from-zero ordering (fir.hpp:138-145)
int ppfg_fir_reference_order(ppfg_plan p, const void* in, uint64_t n_spectra_in, void* out,
                             int mem, void* cuda_stream) {
    PPFG_TRY(check_fir_input(p, in, n_spectra_in, out));
    if (in == out)
        return fail(PPFG_CONFIG_ERROR, "fir: input and output must not alias");
    return run(p, Op::FirRef, in, n_spectra_in, out, mem, cuda_stream, p->T - 1);
}

int ppfg_channelize(ppfg_plan p, const void* in, uint64_t n_rows, void* out, int fft_fallback,
                    int mem, void* cuda_stream) {
    PPFG_TRY(check_plan(p));
    if (n_rows == 0)
        return PPFG_OK;
    if (!in || !out)
        return fail(PPFG_CONFIG_ERROR, "channelize_block: null buffer");
    if (!is_pow2(p->C) && !fft_fallback)
        return fail(PPFG_UNSUPPORTED_SIZE,
                    "channelize_block: non-power-of-two channel count with fallback disabled");
    return run(p, fft_fallback ? Op::Channelize : Op::ChannelizeNoFallback, in, n_rows, out, mem,
               cuda_stream, 0);
}

int ppfg_fir_fft(ppfg_plan p, const void* in, uint64_t n_spectra_in, void* out, int mem,
                 void* cuda_stream) {
    PPFG_TRY(check_fir_input(p, in, n_spectra_in, out));
    if (in == out)
        return fail(PPFG_CONFIG_ERROR, "fir_fft: input and output must not alias");
    return run(p, Op::FirFft, in, n_spectra_in, out, mem, cuda_stream, p->T - 1);
}

int ppfg_mean_power(ppfg_plan p, const void* bins, uint64_t n_spectra, double* mean_power,
                    int mem, void* cuda_stream) {
    PPFG_TRY(check_plan(p));
    if ((n_spectra && !bins) || !mean_power)
        return fail(PPFG_CONFIG_ERROR, "mean_power: null buffer");
    return run_mean_power(p, false, bins, n_spectra, mean_power, mem, cuda_stream);
}

int ppfg_fir_fft_mean_power(ppfg_plan p, const void* in, uint64_t n_spectra_in, double* mean_power,
                            int mem, void* cuda_stream) {
    if (!mean_power)
        return fail(PPFG_CONFIG_ERROR, "fir_fft_mean_power: null output");
    PPFG_TRY(check_fir_input(p, in, n_spectra_in, mean_power));
    return run_mean_power(p, true, in, n_spectra_in, mean_power, mem, cuda_stream);
}

static int one_row(const void* in, uint64_t n, void* out, bool fallback, const char* who) {
    if (n == 0)
        return fail(PPFG_CONFIG_ERROR, std::string(who) + ": empty spectrum");
    if (!fallback && !is_pow2(n))
        return fail(PPFG_UNSUPPORTED_SIZE, "fft: size must be a power of two");
    int dev = 0;
    cudaGetDevice(&dev);
    PlanLease lease;
    PPFG_TRY(lease_plan(n, 0, nullptr, 0, dev, &lease));
    ppfg_plan p = lease.plan;
    int rc;
    if (fallback && is_pow2(n) && n > 1) { // force the naive path for dft_naive
        DeviceGuard dg(p->device);
        void* d = nullptr;
        double2* dr = nullptr;
        rc = cudaMalloc(&d, 2 * n * sizeof(float2)) == cudaSuccess &&
                     cudaMalloc(&dr, n * sizeof(double2)) == cudaSuccess
                 ? PPFG_OK
                 : fail(PPFG_CUDA_ERROR, "dft_naive: device allocation failed");
        if (rc == PPFG_OK) {
            const auto r = host_roots(n);
            // copies on the plan's (non-blocking) stream, so the kernel is
            // ordered after them (a plain cudaMemcpy from pageable memory may
            // return before its DMA has landed)
            cudaMemcpyAsync(dr, r.data(), n * sizeof(double2), cudaMemcpyHostToDevice, p->stream);
            cudaMemcpyAsync(d, in, n * sizeof(float2), cudaMemcpyHostToDevice, p->stream);
            float2* din = static_cast<float2*>(d);
            dft_naive_kernel<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0, p->stream>>>(
                din, din + n, static_cast<unsigned>(n), 1, dr);
            rc = check_launch("dft_naive kernel");
            cudaMemcpyAsync(out, din + n, n * sizeof(float2), cudaMemcpyDeviceToHost, p->stream);
            if (cudaStreamSynchronize(p->stream) != cudaSuccess && rc == PPFG_OK)
                rc = fail(PPFG_CUDA_ERROR, "dft_naive: stream error");
        }
        cudaFree(dr);
        cudaFree(d);
    } else {
        rc = ppfg_channelize(p, in, 1, out, fallback ? 1 : 0, PPFG_MEM_HOST, nullptr);
    }
    return_plan(std::move(lease));
    return rc;
}

int ppfg_fft(const void* in, uint64_t n, void* out) { return one_row(in, n, out, false, "fft"); }
int ppfg_dft_naive(const void* in, uint64_t n, void* out) {
    return one_row(in, n, out, true, "dft_naive");
}

// ---------------------------------------------------------------- shards
int ppfg_shard_range(uint64_t n_spectra_in, uint64_t n_taps, int rank, int world,
                     uint64_t* in_begin, uint64_t* in_count, uint64_t* out_begin,
                     uint64_t* out_count) {
    if (world < 1 || rank < 0 || rank >= world || n_taps == 0)
        return fail(PPFG_CONFIG_ERROR, "shard_range: bad rank/world/taps");
    if (n_spectra_in < n_taps)
        return fail(PPFG_INSUFFICIENT_HISTORY, "fir: need at least n_taps input spectra");
    const uint64_t S_out = n_spectra_in - n_taps + 1;
    const uint64_t base = S_out / world, extra = S_out % world;
    const uint64_t r = static_cast<uint64_t>(rank);
    const uint64_t ob = r * base + std::min<uint64_t>(r, extra);
    const uint64_t oc = base + (r < extra ? 1 : 0);
    *out_begin = ob;
    *out_count = oc;
    *in_begin = ob;
    *in_count = oc > 0 ? oc + n_taps - 1 : 0;
    return PPFG_OK;
}

int ppfg_multi_fir_fft(uint64_t n_channels, uint64_t n_taps, const double* coeff_values,
                       uint32_t flags, const int* devices, int n_devices, const void* host_in,
                       uint64_t n_spectra_in, void* host_out) {
    if (n_devices < 1 || !devices)
        return fail(PPFG_CONFIG_ERROR, "multi_fir_fft: need at least one device");
    if (n_taps == 0 || n_spectra_in < n_taps)
        return fail(n_taps == 0 ? PPFG_CONFIG_ERROR : PPFG_INSUFFICIENT_HISTORY,
                    "fir: need at least n_taps input spectra");
    std::vector<int> status(n_devices, PPFG_OK);
    std::vector<std::string> msgs(n_devices);
    std::vector<std::thread> pool;
    const uint64_t row_bytes = n_channels * sizeof(float2);
    for (int g = 0; g < n_devices; ++g) {
        pool.emplace_back([&, g]() {
            uint64_t ib, ic, ob, oc;
            int st = ppfg_shard_range(n_spectra_in, n_taps, g, n_devices, &ib, &ic, &ob, &oc);
            // per-device plans (and their pinned staging) persist across calls
            PlanLease lease;
            if (st == PPFG_OK && oc > 0)
                st = lease_plan(n_channels, n_taps, coeff_values, flags, devices[g], &lease);
            if (st == PPFG_OK && oc > 0)
                st = ppfg_fir_fft(lease.plan, static_cast<const char*>(host_in) + ib * row_bytes, ic,
                                  static_cast<char*>(host_out) + ob * row_bytes, PPFG_MEM_HOST,
                                  nullptr);
            if (st != PPFG_OK)
                msgs[g] = g_err;
            return_plan(std::move(lease));
            status[g] = st;
        });
    }
    for (auto& t : pool)
        t.join();
    for (int g = 0; g < n_devices; ++g)
        if (status[g] != PPFG_OK)
            return fail(status[g], "shard " + std::to_string(g) + ": " + msgs[g]);
    return PPFG_OK;
}

// Device-resident stream over several GPUs (halo "from peer"):
// segment g lives in d_in[g] on plans[g]'s device with n_taps - 1 spare rows;
// its right edge is completed with the first rows of the following
// segment(s) by cudaMemcpyPeerAsync (NVLink/NVSwitch; a plain device copy when
// both segments share a device), then the fused FIR+FFT runs on the plan's
// stream. No collective; one host thread per segment.
int ppfg_multi_fir_fft_device(const ppfg_plan* plans, int n_segments, void* const* d_in,
                              const uint64_t* seg_rows, void* const* d_out, uint64_t* out_rows) {
    if (n_segments < 1 || !plans || !d_in || !seg_rows || !d_out || !out_rows)
        return fail(PPFG_CONFIG_ERROR, "multi_fir_fft_device: null argument");
    for (int g = 0; g < n_segments; ++g) {
        PPFG_TRY(check_plan(plans[g]));
        if (plans[g]->C != plans[0]->C || plans[g]->T != plans[0]->T || plans[g]->T == 0)
            return fail(PPFG_CONFIG_ERROR, "multi_fir_fft_device: plans differ in C or T");
        if (seg_rows[g] && (!d_in[g] || !d_out[g]))
            return fail(PPFG_CONFIG_ERROR, "multi_fir_fft_device: null segment buffer");
    }
    const uint64_t T = plans[0]->T;
    const uint64_t row_bytes = plans[0]->C * sizeof(float2);
    std::vector<int> status(n_segments, PPFG_OK);
    std::vector<std::string> msgs(n_segments);
    std::vector<std::thread> pool;
    for (int g = 0; g < n_segments; ++g) {
        pool.emplace_back([&, g]() {
            ppfg_plan p = plans[g];
            DeviceGuard dg(p->device);
            auto body = [&]() -> int {
                out_rows[g] = 0;
                if (seg_rows[g] == 0) // an empty segment has no outputs (and may have no buffer)
                    return PPFG_OK;
                // halo: the next T-1 rows of the stream, from the following segment(s)
                uint64_t have = seg_rows[g];
                uint64_t need = T - 1;
                for (int k = g + 1; k < n_segments && need > 0; ++k) {
                    const uint64_t take = std::min<uint64_t>(need, seg_rows[k]);
                    if (take == 0)
                        continue;
                    const int dk = plans[k]->device;
                    if (dk != p->device) {
                        const cudaError_t e = cudaDeviceEnablePeerAccess(dk, 0);
                        if (e == cudaErrorPeerAccessAlreadyEnabled || e == cudaErrorPeerAccessUnsupported)
                            cudaGetLastError(); // copies still work (staged by the driver)
                        else if (e != cudaSuccess)
                            return fail(PPFG_CUDA_ERROR, std::string("peer access: ") + cudaGetErrorString(e));
                    }
                    // the peer segment must be complete: order the copy after
                    // the work queued on its plan's stream (work on other streams
                    // is the caller's to finish, see ppfg.h)
                    cudaEvent_t ready = nullptr;
                    {
                        DeviceGuard pk(dk);
                        PPFG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
                        PPFG_CUDA(cudaEventRecord(ready, plans[k]->stream));
                    }
                    const cudaError_t we = cudaStreamWaitEvent(p->stream, ready, 0);
                    cudaEventDestroy(ready);
                    if (we != cudaSuccess)
                        return fail(PPFG_CUDA_ERROR, std::string("peer halo wait: ") + cudaGetErrorString(we));
                    PPFG_CUDA(cudaMemcpyPeerAsync(static_cast<char*>(d_in[g]) + have * row_bytes, p->device,
                                                  d_in[k], dk, take * row_bytes, p->stream));
                    have += take;
                    need -= take;
                }
                out_rows[g] = have >= T ? have - T + 1 : 0;
                if (out_rows[g] == 0)
                    return PPFG_OK;
                PPFG_TRY(run(p, Op::FirFft, d_in[g], have, d_out[g], PPFG_MEM_DEVICE, nullptr, T - 1));
                PPFG_CUDA(cudaStreamSynchronize(p->stream));
                return PPFG_OK;
            };
            const int st = body();
            if (st != PPFG_OK)
                msgs[g] = g_err;
            status[g] = st;
        });
    }
    for (auto& t : pool)
        t.join();
    for (int g = 0; g < n_segments; ++g)
        if (status[g] != PPFG_OK)
            return fail(status[g], "segment " + std::to_string(g) + ": " + msgs[g]);
    return PPFG_OK;
}

// ----------------------------------------------------------------- synth
int ppfg_synth(uint64_t n_channels, uint64_t seed, uint64_t first_sample, uint64_t n_samples,
               void* out, int mem, int device, void* cuda_stream) {
    if (n_channels == 0)
        return fail(PPFG_CONFIG_ERROR, "synth: n_channels must be >= 1");
    const uint64_t M = 10 * n_channels, f10 = tone_f10(n_channels);
    if (mem == PPFG_MEM_HOST) {
        const auto tone = host_tone(n_channels);
        float2* o = static_cast<float2*>(out);
        for (uint64_t i = 0; i < n_samples; ++i) {
            const uint64_t n = first_sample + i;
            const float2 t = tone[(f10 * n) % M];
            const uint64_t a = splitmix64(seed + (2 * n + 1) * kGolden);
            const uint64_t b = splitmix64(seed + (2 * n + 2) * kGolden);
            volatile float gr = static_cast<float>(irwin_hall4(a)) * kNoiseScale;
            volatile float gi = static_cast<float>(irwin_hall4(b)) * kNoiseScale;
            o[i] = make_float2(t.x + gr, t.y + gi);
        }
        return PPFG_OK;
    }
    DeviceGuard dg(device);
    float2* dtone = nullptr;
    {
        auto& c = tone_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        auto key = std::make_pair(device, n_channels);
        auto it = c.dev.find(key);
        if (it == c.dev.end()) {
            const auto tone = host_tone(n_channels);
            PPFG_CUDA(cudaMalloc(&dtone, tone.size() * sizeof(float2)));
            PPFG_CUDA(cudaMemcpy(dtone, tone.data(), tone.size() * sizeof(float2),
                                 cudaMemcpyHostToDevice));
            // the caller's stream may be non-blocking: the DMA must have landed
            PPFG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
            c.dev[key] = dtone;
        } else {
            dtone = it->second;
        }
    }
    if (n_samples == 0)
        return PPFG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    synth_kernel<<<static_cast<unsigned>(cdiv(n_samples, 256)), 256, 0, st>>>(
        static_cast<float2*>(out), seed, first_sample, n_samples, f10, M, dtone);
    return check_launch("synth kernel");
}

// ------------------------------------------------------- coefficient design
// coeff.hpp:61-144 (same operations as the reference build, incl. the FMA GCC
// contracts 1 - r*r into; pinned against the reference in tests)
static double i0_series(double x) {
    const double y = x * x * 0.25;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 10000; ++k) {
        term *= y / (static_cast<double>(k) * static_cast<double>(k));
        sum += term;
        if (term < sum * 1e-17)
            break;
    }
    return sum;
}

int ppfg_generate_prototype(uint64_t n_channels, uint64_t n_taps, double beta,
                            double cutoff_scale, double* out) {
    if (n_channels == 0 || n_taps == 0)
        return fail(PPFG_CONFIG_ERROR,
                    "generate_prototype: n_channels and n_taps must be >= 1");
    if (!(cutoff_scale > 0.0) || !std::isfinite(cutoff_scale))
        return fail(PPFG_CONFIG_ERROR, "generate_prototype: cutoff_scale must be finite and > 0");
    if (!(beta >= 0.0) || !std::isfinite(beta))
        return fail(PPFG_CONFIG_ERROR, "window beta must be finite and >= 0");
    if (beta > 700.0)
        return fail(PPFG_DOMAIN_ERROR, "bessel_i0: |x| must be <= 700");
    const uint64_t length = n_channels * n_taps;
    std::vector<double> w(length, 1.0);
    if (length > 1 && beta != 0.0) {
        const double denom = i0_series(beta);
        const double span = static_cast<double>(length - 1);
        for (uint64_t k = 0; k < length; ++k) {
            const double r = static_cast<double>(2 * static_cast<int64_t>(k) -
                                                 static_cast<int64_t>(length - 1)) /
                             span;
            w[k] = i0_series(beta * std::sqrt(std::fma(-r, r, 1.0))) / denom;
        }
    }
    const double step = M_PI * cutoff_scale / (2.0 * static_cast<double>(n_channels));
    double sum = 0.0;
    for (uint64_t k = 0; k < length; ++k) {
        const double num = static_cast<double>(2 * static_cast<int64_t>(k) -
                                               static_cast<int64_t>(length - 1));
        const double x = num * step;
        const double v = (x == 0.0 ? 1.0 : std::sin(x) / x) * w[k];
        out[k] = v;
        sum += v;
    }
    if (!std::isfinite(sum) || sum == 0.0)
        return fail(PPFG_DEGENERATE_FILTER, "generate_prototype: coefficient sum vanished");
    for (uint64_t k = 0; k < length; ++k)
        out[k] /= sum;
    return PPFG_OK;
}

} // extern "C"

// ============================================================ streaming
// Device-resident process_stream state (pipeline.hpp:43-200). The carried
// history (carry_history, pipeline.hpp:55-73) stays on the device: each chunk
// of newly completed spectra is uploaded right behind it, the fused kernel
// runs over history ++ chunk, and the last T-1 spectra become the next history
// (ping-pong buffers, no overlap hazards).
// ---------------------------------------------------- pipelined process_stream
// ppfg_process_stream as three concurrent stages (SURVEY §8d host-streamed
// mode): a reader thread pulls blocks of block_spectra*C*8 bytes through the
// read callback into pinned slots (the partial spectrum at a block's end is
// carried into the next slot's prefix); this thread copies each block's whole
// spectra H2D behind the device-resident history (stream s_h2d), runs the fused
// FIR+FFT (plan stream) and copies the spectra back into pinned output slots
// (s_d2h); a writer thread hands them to the write callback in order. Reading,
// PCIe and writing overlap instead of alternating. Byte-identical to the
// reference's loop (pipeline.hpp:89-200): outputs do not depend on the block
// partition, and the byte / sample carry, decode offsets, zero_prime and
// dropped_samples are the same.
namespace {

struct PsShared {
    std::mutex mu;
    std::condition_variable cv;
    bool stop = false; // any stage failed
    int status = PPFG_OK;
    std::string msg;
    uint64_t err_offset = 0;
    void fail_with(int st, const std::string& m, uint64_t off = 0) {
        std::lock_guard<std::mutex> lk(mu);
        if (status == PPFG_OK) {
            status = st;
            msg = m;
            err_offset = off;
        }
        stop = true;
        cv.notify_all();
    }
};

struct PsBlock {
    uint64_t full = 0; // whole spectra in the slot
    int slot = 0;
    bool end = false;
};

int process_stream_pipelined(ppfg_plan p, uint64_t block_spectra, int zero_prime, int fft_fallback,
                             ppfg_read_fn read, void* read_ctx, ppfg_write_fn write, void* write_ctx,
                             ppfg_stream_state* state) {
    constexpr int KH = PsBuffers::KH, KD = PsBuffers::KD, KO = PsBuffers::KO;
    const uint64_t C = p->C, T = p->T;
    const uint64_t row_bytes = C * sizeof(float2);
    if (T == 0)
        return fail(PPFG_CONFIG_ERROR, "config: n_taps must be >= 1");
    if (block_spectra < T) // PpfConfig::validate, pipeline.hpp:33-34
        return fail(PPFG_CONFIG_ERROR, "config: block_spectra must be >= n_taps");
    const uint64_t io = block_spectra * row_bytes; // pipeline.hpp:113
    DeviceGuard dg(p->device);

    PsBuffers* bufs = ps_pool().acquire(p->device);
    struct GiveBack {
        int dev;
        PsBuffers* b;
        ~GiveBack() { ps_pool().give_back(dev, b); }
    } give_back{p->device, bufs};
    if (!bufs->ensure(io, row_bytes, T))
        return fail(PPFG_CUDA_ERROR, "process_stream: buffer allocation failed");
    void* const* h_in = bufs->h_in;
    void* const* h_out = bufs->h_out;
    void* const* d_in = bufs->d_in;
    void* const* d_out = bufs->d_out;
    cudaEvent_t* ev_hin = bufs->ev_hin;
    cudaEvent_t* ev_din = bufs->ev_din;
    cudaEvent_t* ev_comp = bufs->ev_comp;
    cudaEvent_t* ev_d2h = bufs->ev_d2h;

    PsShared sh;
    // reader -> GPU queue (bounded by the KH host slots)
    std::vector<PsBlock> rq;
    size_t rq_head = 0;
    std::vector<uint64_t> hin_released(KH, 0); // blocks whose use of the slot ended
    std::vector<bool> hin_event(KH, false);    // ... with an H2D to wait for
    uint64_t final_carry = 0, final_offset = 0;
    bool read_error = false;
    uint64_t read_error_offset = 0;

    std::thread reader([&]() {
        DeviceGuard rdg(p->device);
        uint64_t carry = 0, offset = 0;
        int prev = -1;
        uint64_t prev_full = 0;
        for (uint64_t blk = 0;; ++blk) {
            const int h = static_cast<int>(blk % KH);
            bool need_sync = false;
            {
                std::unique_lock<std::mutex> lk(sh.mu);
                sh.cv.wait(lk, [&] { return sh.stop || hin_released[h] >= blk / KH; });
                if (sh.stop)
                    return;
                need_sync = blk >= KH && hin_event[h];
            }
            if (need_sync && cudaEventSynchronize(ev_hin[h]) != cudaSuccess) {
                sh.fail_with(PPFG_CUDA_ERROR, "process_stream: H2D failed");
                return;
            }
            char* slot = static_cast<char*>(h_in[h]);
            if (carry)
                std::memcpy(slot, static_cast<char*>(h_in[prev]) + prev_full * row_bytes, carry);
            // a C++ exception must not cross the C-ABI (nor end the process
            // from this thread): a throwing source is a failed read
            int64_t got;
            try {
                got = read(read_ctx, slot + carry, io);
            } catch (...) {
                got = -1;
            }
            bool end = false;
            PsBlock b;
            b.slot = h;
            if (got < 0) { // pipeline.hpp:141-143
                std::lock_guard<std::mutex> lk(sh.mu);
                read_error = true;
                read_error_offset = offset;
                end = true;
            } else if (got == 0) {
                end = true;
            } else {
                offset += static_cast<uint64_t>(got);
                const uint64_t total = carry + static_cast<uint64_t>(got);
                b.full = total / row_bytes;
                carry = total % row_bytes;
                prev = h;
                prev_full = b.full;
                // a short read is not the end: like the reference loop, read
                // again — 0 ends the stream, < 0 is a source failure at the
                // offset after the bytes already delivered (pipeline.hpp:138-143)
            }
            std::lock_guard<std::mutex> lk(sh.mu);
            if (!read_error && got > 0)
                rq.push_back(b);
            if (end) {
                final_carry = carry;
                final_offset = offset;
                PsBlock e;
                e.end = true;
                rq.push_back(e);
                sh.cv.notify_all();
                return;
            }
            sh.cv.notify_all();
        }
    });

    // GPU -> writer queue (bounded by the KO output slots)
    struct WItem {
        int o;
        uint64_t bytes;
        bool end;
    };
    std::vector<WItem> wq;
    size_t wq_head = 0;
    std::vector<uint64_t> out_released(KO, 0);
    std::thread writer([&]() {
        DeviceGuard wdg(p->device);
        for (;;) {
            WItem it;
            {
                std::unique_lock<std::mutex> lk(sh.mu);
                sh.cv.wait(lk, [&] { return sh.stop || wq_head < wq.size(); });
                if (wq_head >= wq.size())
                    return; // stopped
                it = wq[wq_head++];
            }
            if (it.end)
                return;
            if (cudaEventSynchronize(ev_d2h[it.o]) != cudaSuccess) {
                sh.fail_with(PPFG_CUDA_ERROR, "process_stream: D2H failed");
                return;
            }
            int wrc;
            try {
                wrc = it.bytes ? write(write_ctx, h_out[it.o], it.bytes) : 0;
            } catch (...) {
                wrc = 1;
            }
            if (wrc != 0) {
                sh.fail_with(PPFG_IO_ERROR, "process_stream: sink write failed");
                return;
            }
            std::lock_guard<std::mutex> lk(sh.mu);
            ++out_released[it.o];
            sh.cv.notify_all();
        }
    });

    ppfg_stream_state st{};
    cudaStream_t s_h2d = p->s_h2d, s_comp = p->stream, s_d2h = p->s_d2h;
    uint64_t hist = 0;
    if (zero_prime && T > 1) { // pipeline.hpp:110-111
        hist = T - 1;
        cudaMemsetAsync(d_in[0], 0, hist * row_bytes, s_h2d);
    }
    const bool pow2 = is_pow2(C);
    int prev_d = -1;
    uint64_t prev_total = 0, k = 0;
    auto gpu_fail = [&](int rc) {
        sh.fail_with(rc, g_err.empty() ? std::string("process_stream: CUDA error") : g_err, g_err_offset);
    };
    for (;;) {
        PsBlock b;
        {
            std::unique_lock<std::mutex> lk(sh.mu);
            sh.cv.wait(lk, [&] { return sh.stop || rq_head < rq.size(); });
            if (sh.stop)
                break;
            b = rq[rq_head++];
        }
        if (b.end)
            break;
        const int h = b.slot;
        if (b.full == 0) { // nothing whole yet: the carry moves on (pipeline.hpp:177)
            std::lock_guard<std::mutex> lk(sh.mu);
            hin_event[h] = false;
            ++hin_released[h];
            sh.cv.notify_all();
            continue;
        }
        const int d = static_cast<int>(k % KD), o = static_cast<int>(k % KO);
        const uint64_t total = hist + b.full;
        int rc = PPFG_OK;
        // input: slot d is free once block k-KD's kernel has read it
        if (k >= KD && cudaStreamWaitEvent(s_h2d, ev_comp[d], 0) != cudaSuccess)
            rc = fail(PPFG_CUDA_ERROR, "process_stream: stream wait failed");
        if (rc == PPFG_OK && hist && prev_d >= 0 && prev_d != d)
            rc = cudaMemcpyAsync(d_in[d], static_cast<char*>(d_in[prev_d]) + (prev_total - hist) * row_bytes,
                                 hist * row_bytes, cudaMemcpyDeviceToDevice, s_h2d) == cudaSuccess
                     ? PPFG_OK
                     : fail(PPFG_CUDA_ERROR, "process_stream: history copy failed");
        if (rc == PPFG_OK)
            rc = cudaMemcpyAsync(static_cast<char*>(d_in[d]) + hist * row_bytes, h_in[h], b.full * row_bytes,
                                 cudaMemcpyHostToDevice, s_h2d) == cudaSuccess &&
                         cudaEventRecord(ev_hin[h], s_h2d) == cudaSuccess &&
                         cudaEventRecord(ev_din[d], s_h2d) == cudaSuccess
                     ? PPFG_OK
                     : fail(PPFG_CUDA_ERROR, "process_stream: H2D failed");
        {
            std::lock_guard<std::mutex> lk(sh.mu);
            hin_event[h] = true;
            ++hin_released[h];
            sh.cv.notify_all();
        }
        st.bytes_in += b.full * row_bytes;
        const uint64_t n_out = total >= T ? total - T + 1 : 0;
        if (rc == PPFG_OK && n_out) {
            if (!fft_fallback && !pow2)
                rc = fail(PPFG_UNSUPPORTED_SIZE,
                          "channelize_block: non-power-of-two channel count with fallback disabled");
            // output slot o: its previous D2H has been written out by the writer
            if (rc == PPFG_OK) {
                std::unique_lock<std::mutex> lk(sh.mu);
                sh.cv.wait(lk, [&] { return sh.stop || out_released[o] >= k / KO; });
                if (sh.stop)
                    break;
            }
            if (rc == PPFG_OK && (cudaStreamWaitEvent(s_comp, ev_din[d], 0) != cudaSuccess ||
                                  (k >= KO && cudaStreamWaitEvent(s_comp, ev_d2h[o], 0) != cudaSuccess)))
                rc = fail(PPFG_CUDA_ERROR, "process_stream: stream wait failed");
            if (rc == PPFG_OK)
                rc = launch_fir_fft(p, static_cast<const float2*>(d_in[d]), total,
                                    static_cast<float2*>(d_out[o]), s_comp);
            if (rc == PPFG_OK &&
                (cudaEventRecord(ev_comp[d], s_comp) != cudaSuccess ||
                 cudaStreamWaitEvent(s_d2h, ev_comp[d], 0) != cudaSuccess ||
                 cudaMemcpyAsync(h_out[o], d_out[o], n_out * row_bytes, cudaMemcpyDeviceToHost, s_d2h) !=
                     cudaSuccess ||
                 cudaEventRecord(ev_d2h[o], s_d2h) != cudaSuccess))
                rc = fail(PPFG_CUDA_ERROR, "process_stream: D2H failed");
            if (rc == PPFG_OK) {
                std::lock_guard<std::mutex> lk(sh.mu);
                wq.push_back({o, n_out * row_bytes, false});
                sh.cv.notify_all();
            }
        } else if (rc == PPFG_OK) {
            // no output: the slot is still read by the next block's history copy
            // (same stream) and must not be refilled before this block's H2D
            if (cudaEventRecord(ev_comp[d], s_h2d) != cudaSuccess)
                rc = fail(PPFG_CUDA_ERROR, "process_stream: event record failed");
            std::lock_guard<std::mutex> lk(sh.mu);
            ++out_released[o]; // slot o unused by this block
            sh.cv.notify_all();
        }
        if (rc != PPFG_OK) {
            gpu_fail(rc);
            break;
        }
        st.spectra_processed += n_out;
        st.bytes_out += n_out * row_bytes;
        hist = std::min<uint64_t>(T - 1, total); // carry_history (pipeline.hpp:55-73)
        prev_d = d;
        prev_total = total;
        ++k;
    }
    {
        std::lock_guard<std::mutex> lk(sh.mu);
        wq.push_back({0, 0, true});
        sh.cv.notify_all();
    }
    writer.join();
    {
        std::lock_guard<std::mutex> lk(sh.mu);
        sh.stop = true; // release a reader still waiting for a slot
        sh.cv.notify_all();
    }
    reader.join();
    cudaStreamSynchronize(s_h2d);
    cudaStreamSynchronize(s_comp);
    cudaStreamSynchronize(s_d2h);
    int rc = sh.status;
    std::string msg = sh.msg;
    uint64_t off = sh.err_offset;
    if (rc == PPFG_OK && read_error) { // pipeline.hpp:141-143
        rc = PPFG_DECODE_ERROR;
        off = read_error_offset;
        msg = "process_stream: source read failed at byte offset " + std::to_string(off);
    }
    if (rc == PPFG_OK && final_carry % 8 != 0) { // pipeline.hpp:190-192
        rc = PPFG_DECODE_ERROR;
        off = final_offset - final_carry % 8;
        msg = "process_stream: stream truncated mid-sample at byte offset " + std::to_string(off);
    }
    if (rc == PPFG_OK)
        st.dropped_samples += final_carry / 8; // pipeline.hpp:194
    if (state)
        *state = st;
    if (rc != PPFG_OK) {
        g_err_offset = off;
        return fail(rc, msg);
    }
    return PPFG_OK;
}

} // namespace

struct ppfg_stream_s {
    ppfg_plan plan = nullptr;
    uint64_t block_spectra = 0;
    bool fallback = true;
    float2* d_buf[2] = {nullptr, nullptr};
    float2* d_out = nullptr;
    int cur = 0;
    uint64_t cap_rows = 0;  // new rows per device chunk
    uint64_t hist_rows = 0; // valid history rows at the front of d_buf[cur]
    uint8_t byte_carry[8];
    int byte_carry_n = 0;
    std::vector<float2> sample_carry;
    ppfg_stream_state st{};
    uint64_t stream_offset = 0;
};

extern "C" {

int ppfg_stream_open(ppfg_stream* out, ppfg_plan p, uint64_t block_spectra, int zero_prime,
                     int fft_fallback) {
    if (!out)
        return fail(PPFG_CONFIG_ERROR, "stream_open: null stream pointer");
    *out = nullptr;
    PPFG_TRY(check_plan(p));
    if (p->T == 0)
        return fail(PPFG_CONFIG_ERROR, "config: n_taps must be >= 1");
    if (block_spectra < p->T) // PpfConfig::validate, pipeline.hpp:33-34
        return fail(PPFG_CONFIG_ERROR, "config: block_spectra must be >= n_taps");
    DeviceGuard dg(p->device);
    auto* s = new ppfg_stream_s();
    s->plan = p;
    s->block_spectra = block_spectra;
    s->fallback = fft_fallback != 0;
    const uint64_t row_bytes = p->C * sizeof(float2);
    s->cap_rows = std::max<uint64_t>(1, std::min<uint64_t>(block_spectra, kChunkBytes / row_bytes));
    const uint64_t buf_rows = s->cap_rows + p->T;
    for (int i = 0; i < 2; ++i) {
        if (cudaMalloc(&s->d_buf[i], buf_rows * row_bytes) != cudaSuccess) {
            ppfg_stream_destroy(s);
            return fail(PPFG_CUDA_ERROR, "stream_open: device allocation failed");
        }
    }
    if (cudaMalloc(&s->d_out, buf_rows * row_bytes) != cudaSuccess) {
        ppfg_stream_destroy(s);
        return fail(PPFG_CUDA_ERROR, "stream_open: device allocation failed");
    }
    if (zero_prime) { // pipeline.hpp:110-111
        s->hist_rows = p->T - 1;
        if (s->hist_rows &&
            cudaMemsetAsync(s->d_buf[0], 0, s->hist_rows * row_bytes, p->stream) != cudaSuccess) {
            ppfg_stream_destroy(s);
            return fail(PPFG_CUDA_ERROR, "stream_open: history priming failed");
        }
    }
    *out = s;
    return PPFG_OK;
}

int ppfg_stream_push(ppfg_stream s, const void* bytes, uint64_t n, void* out, uint64_t out_cap,
                     uint64_t* out_len) {
    if (!s)
        return fail(PPFG_CONFIG_ERROR, "stream_push: null stream");
    ppfg_plan p = s->plan;
    DeviceGuard dg(p->device);
    const uint64_t C = p->C, T = p->T;
    const uint64_t row_bytes = C * sizeof(float2);
    *out_len = 0;
    const uint8_t* data = static_cast<const uint8_t*>(bytes);
    uint64_t avail = n;
    // complete a sample split across pushes (pipeline.hpp:151-163)
    if (s->byte_carry_n != 0 && avail) {
        const uint64_t take = std::min<uint64_t>(8 - s->byte_carry_n, avail);
        std::memcpy(s->byte_carry + s->byte_carry_n, data, take);
        s->byte_carry_n += static_cast<int>(take);
        data += take;
        avail -= take;
        if (s->byte_carry_n == 8) {
            float2 z;
            std::memcpy(&z, s->byte_carry, 8);
            s->sample_carry.push_back(z);
            s->byte_carry_n = 0;
        }
    }
    // append bytes to the sample / byte carry (pipeline.hpp:165-172)
    auto carry_bytes = [&](const uint8_t* d, uint64_t k) {
        const uint64_t full = k / 8, tail = k % 8;
        const size_t old = s->sample_carry.size();
        s->sample_carry.resize(old + full);
        std::memcpy(s->sample_carry.data() + old, d, full * 8);
        if (tail) {
            std::memcpy(s->byte_carry, d + full * 8, tail);
            s->byte_carry_n = static_cast<int>(tail);
        }
    };
    s->stream_offset += n;
    // nothing carried: whole spectra go to the device straight from the
    // caller's buffer (a DMA when it is pinned), only the tail is carried
    const bool direct = s->sample_carry.empty() && s->byte_carry_n == 0;
    const float2* src;
    uint64_t full_spectra;
    if (direct) {
        full_spectra = avail / row_bytes;
        src = reinterpret_cast<const float2*>(data);
    } else {
        carry_bytes(data, avail);
        full_spectra = s->sample_carry.size() / C;
        src = s->sample_carry.data();
    }
    uint64_t done = 0;
    char* o = static_cast<char*>(out);
    while (done < full_spectra) {
        const uint64_t rows = std::min(s->cap_rows, full_spectra - done);
        float2* buf = s->d_buf[s->cur];
        PPFG_CUDA(cudaMemcpyAsync(buf + s->hist_rows * C, src + done * C, rows * row_bytes,
                                  cudaMemcpyHostToDevice, p->stream));
        const uint64_t total = s->hist_rows + rows;
        s->st.bytes_in += rows * row_bytes;
        if (total >= T) {
            const uint64_t n_out = total - T + 1;
            if (*out_len + n_out * row_bytes > out_cap)
                return fail(PPFG_CONFIG_ERROR, "stream_push: output buffer too small");
            if (s->fallback || is_pow2(C)) {
                PPFG_TRY(launch_fir_fft(p, buf, total, s->d_out, p->stream));
            } else {
                return fail(PPFG_UNSUPPORTED_SIZE, "channelize_block: non-power-of-two channel "
                                                   "count with fallback disabled");
            }
            PPFG_CUDA(cudaMemcpyAsync(o + *out_len, s->d_out, n_out * row_bytes,
                                      cudaMemcpyDeviceToHost, p->stream));
            *out_len += n_out * row_bytes;
            s->st.spectra_processed += n_out;
            s->st.bytes_out += n_out * row_bytes;
        }
        const uint64_t keep = std::min<uint64_t>(T - 1, total);
        if (keep)
            PPFG_CUDA(cudaMemcpyAsync(s->d_buf[s->cur ^ 1], buf + (total - keep) * C,
                                      keep * row_bytes, cudaMemcpyDeviceToDevice, p->stream));
        s->cur ^= 1;
        s->hist_rows = keep;
        done += rows;
    }
    if (direct)
        carry_bytes(data + full_spectra * row_bytes, avail - full_spectra * row_bytes);
    else
        s->sample_carry.erase(s->sample_carry.begin(),
                              s->sample_carry.begin() + static_cast<std::ptrdiff_t>(done * C));
    PPFG_CUDA(cudaStreamSynchronize(p->stream));
    return PPFG_OK;
}

int ppfg_stream_close(ppfg_stream s, ppfg_stream_state* state) {
    if (!s)
        return fail(PPFG_CONFIG_ERROR, "stream_close: null stream");
    if (s->byte_carry_n != 0) { // pipeline.hpp:190-192
        g_err_offset = s->stream_offset - s->byte_carry_n;
        const std::string m = "process_stream: stream truncated mid-sample at byte offset " +
                              std::to_string(g_err_offset);
        if (state)
            *state = s->st;
        return fail(PPFG_DECODE_ERROR, m);
    }
    s->st.dropped_samples += s->sample_carry.size(); // pipeline.hpp:194
    s->sample_carry.clear();
    if (state)
        *state = s->st;
    return PPFG_OK;
}

int ppfg_stream_destroy(ppfg_stream s) {
    if (!s)
        return PPFG_OK;
    DeviceGuard dg(s->plan->device);
    cudaFree(s->d_buf[0]);
    cudaFree(s->d_buf[1]);
    cudaFree(s->d_out);
    delete s;
    return PPFG_OK;
}

int ppfg_process_stream(ppfg_plan p, uint64_t block_spectra, int zero_prime, int fft_fallback,
                        ppfg_read_fn read, void* read_ctx, ppfg_write_fn write, void* write_ctx,
                        ppfg_stream_state* state) {
    if (state)
        *state = ppfg_stream_state{};
    PPFG_TRY(check_plan(p));
    if (!read || !write)
        return fail(PPFG_CONFIG_ERROR, "process_stream: null callback");
    return process_stream_pipelined(p, block_spectra, zero_prime, fft_fallback, read, read_ctx, write,
                                    write_ctx, state);
}

} // extern "C"

// ========================================================= device memory
extern "C" {

int ppfg_device_alloc(void** ptr, uint64_t bytes, int device) {
    if (!ptr)
        return fail(PPFG_CONFIG_ERROR, "device_alloc: null pointer");
    *ptr = nullptr;
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess)
        return fail(PPFG_NO_DEVICE, "ppfg: no current device");
    DeviceGuard dg(device);
    PPFG_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
    return PPFG_OK;
}

int ppfg_device_free(void* ptr) {
    if (ptr)
        PPFG_CUDA(cudaFree(ptr));
    return PPFG_OK;
}

int ppfg_memcpy(void* dst, const void* src, uint64_t bytes) {
    if (bytes) {
        PPFG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
        // complete on return (a copy from pageable memory may return before
        // its DMA lands; the plans' kernels run on non-blocking streams)
        PPFG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
    return PPFG_OK;
}

int ppfg_plan_synchronize(ppfg_plan p) {
    PPFG_TRY(check_plan(p));
    DeviceGuard dg(p->device);
    PPFG_CUDA(cudaStreamSynchronize(p->stream));
    return PPFG_OK;
}

} // extern "C"

#ifdef PPFG_TRACE
extern "C" int ppfg_debug_trace(unsigned long long* out) {
    PPFG_CUDA(cudaMemcpyFromSymbol(out, ppfg::g_trace, sizeof(ppfg::g_trace)));
    return PPFG_OK;
}
#endif
