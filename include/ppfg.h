/*
 * ppfg.h — C-ABI of the B200-native polyphase filter bank (libppfg.so).
 *
 * Plain pointers, sizes and status codes; no C++ or torch types. Every entry
 * point below replaces one function of the reference's header-only C++ API
 * (/root/reference/proj/include/ppf/, cited file:line); include/ppf_gpu/ppf.hpp
 * wraps these back into the reference's value types and exception classes so
 * reference callers switch by changing an include path and a namespace.
 *
 * Data layout (identical to the reference): complex samples are interleaved
 * float32 pairs (std::complex<float>); a block is spectrum-major, sample n is
 * spectrum n / C, channel n % C (fir.hpp:22-38). Coefficients are tap-major
 * doubles values[t*C + c] (coeff.hpp:50-58), quantized to float32 inside the
 * plan exactly as quantize_taps does (fir.hpp:69-74).
 *
 * Memory kinds: PPFG_MEM_DEVICE calls take device pointers, enqueue on the
 * given cudaStream_t (NULL = the plan's own non-blocking stream; pass
 * cudaStreamLegacy, (void*)1, for the legacy default stream) and return
 * without synchronising. PPFG_MEM_HOST calls take host pointers (pinned or pageable),
 * run a chunked H2D -> kernel -> D2H pipeline and return when the output is in
 * host memory (the reference's synchronous contract, fir.hpp:158).
 *
 * Threading: calls on different plans are reentrant; a plan must not be used
 * by two host threads at once (it owns its staging buffers and streams).
 * Errors: every function returns a ppfg_status; ppfg_last_error() holds the
 * message of the calling thread's last failure.
 */
#ifndef PPFG_H
#define PPFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One code per class of include/ppf/errors.hpp (1..6), plus the device. */
typedef enum {
    PPFG_OK = 0,
    PPFG_CONFIG_ERROR = 1,             /* ppf::config_error            errors.hpp:11-13 */
    PPFG_INSUFFICIENT_HISTORY = 2,     /* ppf::insufficient_history_error errors.hpp:16-18 */
    PPFG_UNSUPPORTED_SIZE = 3,         /* ppf::unsupported_size_error  errors.hpp:21-23 */
    PPFG_DEGENERATE_FILTER = 4,        /* ppf::degenerate_filter_error errors.hpp:26-28 */
    PPFG_DECODE_ERROR = 5,             /* ppf::decode_error{byte_offset} errors.hpp:32-38 */
    PPFG_IO_ERROR = 6,                 /* ppf::io_error                errors.hpp:41-43 */
    PPFG_CUDA_ERROR = 7,               /* a CUDA runtime/launch failure */
    PPFG_NO_DEVICE = 8,                /* no usable sm_100 device */
    PPFG_DOMAIN_ERROR = 9              /* std::domain_error (bessel_i0, metrics) */
} ppfg_status;

typedef enum { PPFG_MEM_HOST = 0, PPFG_MEM_DEVICE = 1 } ppfg_mem;

/* Plan flags. The default (0) is PPFG_EXACT: FIR accumulates in FP64 in the
 * reference's per-output operation order and the FFT runs the reference's
 * radix-2 butterflies on its float32 twiddle table, so every output is
 * bit-identical to ppf_fir_optimized / channelize_block. PPFG_FAST lets the
 * fused FIR+FFT kernel accumulate the FIR in FP32 (max|err|/RMS well inside the
 * north-star 1e-5*log2(C) bound; FIR-only calls stay exact). PPFG_UNFUSED
 * forces FIR -> HBM -> FFT even where a fused kernel exists (for comparison).
 * PPFG_CLUSTER also admits the thread-block-cluster fused kernels that are
 * not taken by default (C = 8192); the others (C = 2048, 4096; T = 16, 32 at
 * C = 1024; FP64 at C = 1024, 2048) are used whenever they apply, since they
 * measured faster than the unfused path. */
enum {
    PPFG_EXACT = 0u,
    PPFG_FAST = 1u,
    PPFG_UNFUSED = 2u,
    PPFG_CLUSTER = 4u,
    PPFG_K1_PREFETCH = 8u, /* comparison only: FIR-only kernel with register prefetch
                              instead of TMA-staged input (same results) */
    PPFG_FIR_LEGACY = 16u, /* comparison only: the lane-window FIR kernels (K1/K1t/K1f)
                              instead of the register-blocked K1b for T >= 16 */
    PPFG_L2X = 32u         /* also admit the L2-exchange fused kernels (K7, l2x.cuh)
                              that are not taken by default */
};

typedef struct ppfg_plan_s* ppfg_plan;
typedef struct ppfg_stream_s* ppfg_stream;

/* Streaming state; mirrors ppf::StreamState (pipeline.hpp:43-49). */
typedef struct {
    uint64_t spectra_processed;
    uint64_t bytes_in;
    uint64_t bytes_out;
    uint64_t dropped_samples;
} ppfg_stream_state;

/* ---- plans ---------------------------------------------------------------- */

/* Build the device-side state for a (C, T) channelizer: f32 taps
 * (quantize_taps, fir.hpp:69-74), the FFT twiddle table of FftPlan
 * (dft.hpp:88-98, computed on the host in double exactly as the reference
 * does) and, for non-power-of-two C, the dft_naive root table (dft.hpp:47-51).
 * coeff_values may be NULL when n_taps == 0 (an FFT-only plan for
 * channelize_block). Validation mirrors check_fir_preconditions
 * (fir.hpp:56-65): n_channels >= 1, coefficient count == C*T. device = -1
 * selects the calling thread's current CUDA device. */
int ppfg_plan_create(ppfg_plan* plan, uint64_t n_channels, uint64_t n_taps,
                     const double* coeff_values, uint32_t flags, int device);
int ppfg_plan_destroy(ppfg_plan plan);
/* The plan's own CUDA stream (as void*). */
void* ppfg_plan_stream(ppfg_plan plan);

/* ---- the hot path --------------------------------------------------------- */

/* ppf_fir_optimized (fir.hpp:158-212) and ppf_fir_reference (fir.hpp:123-151):
 * out[s][c] = sum_t h[t][c] * in[s+t][c] for s < n_spectra_in - T + 1, FP64
 * accumulation in ascending t, rounded to f32. Bit-identical to the reference.
 * Errors: INSUFFICIENT_HISTORY if n_spectra_in < T (fir.hpp:63-64). */
int ppfg_fir(ppfg_plan plan, const void* in, uint64_t n_spectra_in, void* out, int mem,
             void* cuda_stream);

/* ppf_fir_reference (fir.hpp:123-151): same as ppfg_fir except that the first
 * tap starts from fma(h, x, 0.0) rather than the product h*x; the two differ
 * only in the sign of outputs that are exactly zero. */
int ppfg_fir_reference_order(ppfg_plan plan, const void* in, uint64_t n_spectra_in, void* out,
                             int mem, void* cuda_stream);

/* channelize_block (dft.hpp:175-235): C-point forward DFT of each of n_rows
 * rows, natural order, unnormalised. Power-of-two C: the reference radix-2
 * DIT (FftPlan::transform, dft.hpp:105-148), bit-identical. Otherwise
 * dft_naive (dft.hpp:39-66) when fft_fallback, else UNSUPPORTED_SIZE.
 * n_rows == 0 is a no-op (dft.hpp:187-188). in == out is allowed. */
int ppfg_channelize(ppfg_plan plan, const void* in, uint64_t n_rows, void* out,
                    int fft_fallback, int mem, void* cuda_stream);

/* The fused hot path: channelize_block(ppf_fir_optimized(in)) as composed at
 * pipeline.hpp:125-127, without the intermediate HBM round trip where a fused
 * kernel exists for (C, T). Output n_spectra_in - T + 1 rows. */
int ppfg_fir_fft(ppfg_plan plan, const void* in, uint64_t n_spectra_in, void* out, int mem,
                 void* cuda_stream);

/* Downstream detection, the step after channelization: per-channel mean power
 * as `ppf inspect` computes it (cmd_inspect, cli.hpp:307-317):
 *   mean_power[c] = sum_s ((double)re^2 + (double)im^2) / n_spectra
 * over n_spectra rows of channelized bins (ppfg_mean_power) or over the
 * n_spectra_in - T + 1 output spectra of ppfg_fir_fft (ppfg_fir_fft_mean_power;
 * where a fused kernel exists the bins never reach memory, so the pass only
 * reads its input). mean_power holds C doubles, in the same memory kind as
 * the input. Each power term is exact as in the reference; the sum is taken
 * per CTA in spectrum order and then over CTAs in a fixed order, so results
 * are deterministic and differ from the reference's single running sum only
 * by summation order (relative error ~1e-15). n_spectra == 0 gives zeros
 * (the reference prints no mean then). */
int ppfg_mean_power(ppfg_plan plan, const void* bins, uint64_t n_spectra, double* mean_power,
                    int mem, void* cuda_stream);
int ppfg_fir_fft_mean_power(ppfg_plan plan, const void* in, uint64_t n_spectra_in,
                            double* mean_power, int mem, void* cuda_stream);

/* Which kernel ppfg_fir_fft will run for this plan: 0 = unfused FIR+FFT,
 * 1 = fused FP32-FIR, 2 = fused FP64 (bit-exact) FIR, 3 / 4 = the cluster
 * versions of 1 / 2, 5 / 6 = the warp-level tiny-C (1..32) versions of 1 / 2,
 * 7 / 8 = the L2-exchange versions (K7) of 1 / 2. */
int ppfg_fir_fft_kind(ppfg_plan plan);
/* The kernel ppfg_fir_fft launches for this plan, named the way ncu prints it
 * ("fused_fir_fft_kernel<FusedCfg<10, 8, 2, 0, ...>>"), so measurements can be
 * matched to profiles of exactly that kernel. Valid while the plan lives. */
const char* ppfg_fir_fft_kernel_name(ppfg_plan plan);

/* The device's theoretical HBM bandwidth in GB/s (2 x memory clock x bus
 * width; device -1 = the current one): the default roofline denominator of
 * the report layer (BenchmarkReport::roofline_frac). */
int ppfg_device_hbm_gbs(int device, double* gb_per_sec);

/* Host memcpy split over the library's small pool of copy threads (the same
 * pool that stages pageable buffers for the host-memory entry points): for
 * the drop-in's host-side bookkeeping (carry_history, pipeline.hpp:55-73). */
int ppfg_host_copy(void* dst, const void* src, uint64_t bytes);
/* The calling thread's current CUDA device (plan caches key on it). */
int ppfg_current_device(int* device);

/* ---- single-row helpers (dft.hpp:39-66, 160-169), host memory ------------- */
int ppfg_fft(const void* in, uint64_t n, void* out);        /* UNSUPPORTED_SIZE if n not 2^k */
int ppfg_dft_naive(const void* in, uint64_t n, void* out);

/* ---- streaming (pipeline.hpp:55-200) --------------------------------------- */

/* A device-resident equivalent of process_stream's state: the (T-1)-spectrum
 * history (carry_history, pipeline.hpp:55-73) lives on the device, input is
 * pushed as raw little-endian f32 pairs in arbitrary byte counts (partial
 * samples and spectra are carried, pipeline.hpp:150-184), and every complete
 * spectrum is channelized once its window is complete. Output bytes are
 * independent of how the input is split. */
int ppfg_stream_open(ppfg_stream* stream, ppfg_plan plan, uint64_t block_spectra, int zero_prime,
                     int fft_fallback);
/* Push n bytes; writes the newly completed output spectra to out (host
 * memory, capacity out_cap bytes; need at most
 * (n/(8*C) + 2 + block_spectra) * 8*C) and their byte count to *out_len. */
int ppfg_stream_push(ppfg_stream stream, const void* bytes, uint64_t n, void* out,
                     uint64_t out_cap, uint64_t* out_len);
/* End of input: DECODE_ERROR (offset in ppfg_last_error_offset) when the
 * stream ended mid-sample (pipeline.hpp:190-192); trailing samples of an
 * incomplete spectrum are counted in dropped_samples (pipeline.hpp:194). */
int ppfg_stream_close(ppfg_stream stream, ppfg_stream_state* state);
int ppfg_stream_destroy(ppfg_stream stream);

/* process_stream (pipeline.hpp:89-200) over caller callbacks. read returns
 * the number of bytes produced (any count <= n; it is called again until it
 * returns 0 = end of input, or < 0 = source failure -> DECODE_ERROR at the
 * offset after the bytes already delivered, pipeline.hpp:138-143); write
 * returns 0 on success (non-zero -> IO_ERROR, pipeline.hpp:131-132). The
 * callbacks run on library threads; they must not let C++ exceptions escape
 * (one that does is treated as a failed read / write). */
typedef int64_t (*ppfg_read_fn)(void* ctx, void* buf, uint64_t n);
typedef int (*ppfg_write_fn)(void* ctx, const void* buf, uint64_t n);
int ppfg_process_stream(ppfg_plan plan, uint64_t block_spectra, int zero_prime, int fft_fallback,
                        ppfg_read_fn read, void* read_ctx, ppfg_write_fn write, void* write_ctx,
                        ppfg_stream_state* state);

/* ---- multi-GPU sharding ----------------------------------------- */

/* Split the output spectra [0, S_out) into `world` contiguous ranges; shard
 * `rank` reads input spectra [*in_begin, *in_begin + *in_count) — its own
 * segment plus the (T-1)-spectrum halo at its right edge — and writes output
 * spectra [*out_begin, *out_begin + *out_count). No collective is needed. */
int ppfg_shard_range(uint64_t n_spectra_in, uint64_t n_taps, int rank, int world,
                     uint64_t* in_begin, uint64_t* in_count, uint64_t* out_begin,
                     uint64_t* out_count);
/* Run ppfg_fir_fft over host buffers on n_devices GPUs at once, one host
 * thread per device, each on its shard with its halo. */
int ppfg_multi_fir_fft(uint64_t n_channels, uint64_t n_taps, const double* coeff_values,
                       uint32_t flags, const int* devices, int n_devices, const void* host_in,
                       uint64_t n_spectra_in, void* host_out);

/* Device-resident stream distributed over GPUs (the halo read from
 * the peer): segment g holds the next seg_rows[g] input spectra of one stream in
 * d_in[g], on plans[g]'s device, in a buffer with room for seg_rows[g] +
 * n_taps - 1 spectra. Each segment's right edge is completed with the first
 * n_taps - 1 spectra of the following segment(s) by cudaMemcpyPeerAsync over
 * NVLink/NVSwitch, then the fused FIR+FFT (ppfg_fir_fft) writes out_rows[g] =
 * (seg_rows[g] + halo) - n_taps + 1 output spectra to d_out[g] — the stream's
 * outputs in order, byte-identical to one ppfg_fir_fft over the whole stream.
 * Plans share C and T; one host thread per segment; returns when all are done.
 * Every segment's input must be complete when this is called: work queued on
 * the plans' own streams is waited for, work on any other stream is the
 * caller's to synchronise. An empty segment (seg_rows[g] == 0) may pass null
 * buffers and gets out_rows[g] = 0.
 * Replaces the multi-worker one-shot of ppf_fir_optimized/channelize_block
 * (fir.hpp:158-212, dft.hpp:175-235) when the stream is sharded across GPUs. */
int ppfg_multi_fir_fft_device(const ppfg_plan* plans, int n_segments, void* const* d_in,
                              const uint64_t* seg_rows, void* const* d_out, uint64_t* out_rows);

/* ---- synthetic input --------------------------------------------- */

/* Counter-based tone + noise: x[n] = e^{2 pi i f n / C} + (g1 + i g2) with
 * f = C/8 + 0.3 bins (exact integer phase reduction, float32 phase table built
 * on the host) and g from splitmix64(seed, n) (Irwin-Hall, 4 x 16-bit). Same
 * bytes on host and device; sample index n starts at first_sample so shards
 * generate their own segment with no communication. */
int ppfg_synth(uint64_t n_channels, uint64_t seed, uint64_t first_sample, uint64_t n_samples,
               void* out, int mem, int device, void* cuda_stream);

/* ---- coefficient design (coeff.hpp:61-144) ------------------------------------ */
int ppfg_generate_prototype(uint64_t n_channels, uint64_t n_taps, double beta,
                            double cutoff_scale, double* out);

/* ---- metrics (bench.hpp:25-36, fir.hpp:49-52, dft.hpp:28-35) ----------------- */
uint64_t ppfg_flops_for_fir(uint64_t n_channels, uint64_t n_taps, uint64_t n_spectra_out);
uint64_t ppfg_flops_for_dft(uint64_t n_channels, uint64_t n_spectra);

/* ---- device memory (for callers without their own CUDA runtime) --------------- */
/* device = -1: the calling thread's current device. ppfg_memcpy infers the
 * direction from the pointers (unified addressing) and is synchronous. */
int ppfg_device_alloc(void** ptr, uint64_t bytes, int device);
int ppfg_device_free(void* ptr);
int ppfg_memcpy(void* dst, const void* src, uint64_t bytes);
/* Wait for everything enqueued on the plan's stream. */
int ppfg_plan_synchronize(ppfg_plan plan);

/* ---- diagnostics --------------------------------------------------------------- */
const char* ppfg_last_error(void);
uint64_t ppfg_last_error_offset(void);
/* Number of kernels this library has launched in this process (all devices). */
uint64_t ppfg_kernel_launches(void);
const char* ppfg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PPFG_H */
