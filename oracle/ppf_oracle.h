/*
 * ppf_oracle.h — CPU restatement of the reference polyphase filter bank path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_1411_3656_b200/,
 * include/) links or calls this. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker or as the timed CPU baseline.
 *
 * Every function restates the reference algorithm in plain C and cites the
 * reference file:line it follows (paths relative to /root/reference/proj/).
 * Parity of this restatement is pinned (tests/test_oracle.py) against:
 *   - the reference itself compiled from its own headers (oracle/_ref, built
 *     by oracle/Makefile from /root/reference) — bit-for-bit;
 *   - golden vectors generated from that build (tests/golden/reference_vectors.npz, script
 *     tests/golden/make_golden.py);
 *   - the known-answer values the reference tests hard-code.
 *
 * Data layout everywhere: complex samples are interleaved float pairs
 * (re, im) == std::complex<float>; sample n is spectrum n / C, channel n % C
 * (include/ppf/fir.hpp:22-38). Coefficients are tap-major doubles,
 * values[t*C + c] (include/ppf/coeff.hpp:50-58).
 */
#ifndef PPF_ORACLE_H
#define PPF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: identical numbering to include/ppfg.h */
enum {
    PPFO_OK = 0,
    PPFO_CONFIG_ERROR = 1,
    PPFO_INSUFFICIENT_HISTORY = 2,
    PPFO_UNSUPPORTED_SIZE = 3,
    PPFO_DEGENERATE_FILTER = 4,
    PPFO_DECODE_ERROR = 5,
    PPFO_IO_ERROR = 6,
    PPFO_DOMAIN_ERROR = 9,
    PPFO_OTHER = 99
};

/* coeff.hpp:61-65 */
double ppfo_sinc(double x);
/* coeff.hpp:69-82; returns NaN-free value, *status = PPFO_DOMAIN_ERROR past 700 */
double ppfo_bessel_i0(double x, int* status);
/* coeff.hpp:87-104 */
int ppfo_kaiser_window(size_t length, double beta, double* out);
/* coeff.hpp:110-144; out has C*T doubles */
int ppfo_generate_prototype(size_t n_channels, size_t n_taps, double beta, double cutoff_scale,
                            double* out);

/* fir.hpp:49-52 and dft.hpp:28-35 */
uint64_t ppfo_flops_for_fir(size_t n_channels, size_t n_taps, size_t n_spectra_out);
uint64_t ppfo_flops_for_dft(size_t n_channels, size_t n_spectra);

/* fir.hpp:158-212 (+85-110). Output spectra = n_spectra_in - n_taps + 1.
 * reference_order != 0 reproduces fir.hpp:123-151 instead (fma from 0.0 at
 * t = 0; differs from the optimized order only in the sign of exact zeros). */
int ppfo_fir(const float* in, size_t n_spectra_in, size_t n_channels, size_t n_taps,
             const double* coeff_values, float* out, int reference_order);

/* dft.hpp:39-66 (single row, n >= 1) */
int ppfo_dft_naive(const float* in, size_t n, float* out);
/* dft.hpp:72-148 + 160-169: radix-2 DIT on one row, in place */
int ppfo_fft(float* row, size_t n);
/* dft.hpp:175-235 */
int ppfo_channelize(const float* filtered, size_t n_rows, size_t n_channels, int fft_fallback,
                    float* out);
/* fir then channelize, as composed at pipeline.hpp:125-127 */
int ppfo_fir_fft(const float* in, size_t n_spectra_in, size_t n_channels, size_t n_taps,
                 const double* coeff_values, int fft_fallback, float* out);

/* cmd_inspect's mean power (cli.hpp:307-317): mean[c] = sum over spectra
 * (in order, one running double sum per channel) of
 * (double)re*re + (double)im*im, divided by n_spectra (left 0 when
 * n_spectra == 0). */
int ppfo_mean_power(const float* bins, size_t n_spectra, size_t n_channels, double* mean);

/* pipeline.hpp:89-200 over an in-memory byte source. The source is read in
 * requests of block_spectra*C*8 bytes, each satisfied in full until EOF
 * (istringstream semantics). `out` must hold at least
 * (src_len / (8*C) + n_taps) * C * 8 bytes. */
typedef struct {
    uint64_t spectra_processed;
    uint64_t bytes_in;
    uint64_t bytes_out;
    uint64_t dropped_samples;
    uint64_t error_offset; /* byte offset for PPFO_DECODE_ERROR */
} ppfo_stream_state;

int ppfo_process_stream(size_t n_channels, size_t n_taps, size_t block_spectra, int fft_fallback,
                        int zero_prime, const double* coeff_values, const uint8_t* src,
                        size_t src_len, uint8_t* out, ppfo_stream_state* state);

/* The bench's synthetic workload (not a reference function):
 * x[n] = tone[(f10*n) mod 10C] + (g_re + i g_im), tone = f32 e^{2 pi i k/(10C)},
 * f10 = 10C/8 + 3, g = Irwin-Hall(4 x 16 bit of splitmix64(seed + (2n+1|2n+2)
 * * golden))) * 2.64293e-05f. Integer + IEEE-rounded float ops only, so the
 * bytes equal the product's device generator (libppfg ppfg_synth); used to
 * feed the reference's CPU arm without loading the product library. */
int ppfo_synth(size_t n_channels, uint64_t seed, uint64_t first_sample, size_t n_samples,
               float* out);

#ifdef __cplusplus
}
#endif
#endif
