/*
 * ppf_oracle.c — CPU restatement of the reference PPF path (FIR + FFT +
 * streaming carry). TEST INFRASTRUCTURE ONLY: see ppf_oracle.h.
 *
 * Compiled with -ffp-contract=off: every fused multiply-add below is written
 * out explicitly (fma()) exactly where the reference either calls std::fma or
 * where GCC contracts the reference expression when the reference is built
 * the way its CMakeLists builds it (-std=gnu++20 -O3 -march=native on an
 * FMA-capable x86 host; proj/CMakeLists.txt:4-27). The contraction sites are
 * marked "[contract]" and pinned bit-for-bit against oracle/_ref in
 * tests/test_oracle.py.
 *
 * File:line citations are relative to /root/reference/proj/.
 */
#include "ppf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- coeff */

/* include/ppf/coeff.hpp:61-65 */
double ppfo_sinc(double x) {
    if (x == 0.0)
        return 1.0;
    return sin(x) / x;
}

/* include/ppf/coeff.hpp:69-82 (power series, 1e-17 relative stop) */
double ppfo_bessel_i0(double x, int* status) {
    if (!(fabs(x) <= 700.0)) {
        if (status)
            *status = PPFO_DOMAIN_ERROR;
        return 0.0;
    }
    const double y = x * x * 0.25;
    double term = 1.0;
    double sum = 1.0;
    for (int k = 1; k < 10000; ++k) {
        term *= y / ((double)k * (double)k);
        sum += term;
        if (term < sum * 1e-17)
            break;
    }
    return sum;
}

/* include/ppf/coeff.hpp:87-104 */
int ppfo_kaiser_window(size_t length, double beta, double* w) {
    if (length == 0)
        return PPFO_CONFIG_ERROR;
    if (!(beta >= 0.0) || !isfinite(beta))
        return PPFO_CONFIG_ERROR;
    for (size_t k = 0; k < length; ++k)
        w[k] = 1.0;
    if (length == 1 || beta == 0.0)
        return PPFO_OK;
    int st = PPFO_OK;
    const double denom = ppfo_bessel_i0(beta, &st);
    if (st != PPFO_OK)
        return st;
    const double span = (double)(length - 1);
    for (size_t k = 0; k < length; ++k) {
        const double r = (double)(2 * (int64_t)k - (int64_t)(length - 1)) / span;
        /* [contract] 1.0 - r*r  ->  fma(-r, r, 1.0) (coeff.hpp:100) */
        w[k] = ppfo_bessel_i0(beta * sqrt(fma(-r, r, 1.0)), &st) / denom;
        if (st != PPFO_OK)
            return st;
    }
    return PPFO_OK;
}

/* include/ppf/coeff.hpp:110-144, default cutoff scale 1.5 (coeff.hpp:24) */
int ppfo_generate_prototype(size_t n_channels, size_t n_taps, double beta, double cutoff_scale,
                            double* out) {
    if (n_channels == 0 || n_taps == 0)
        return PPFO_CONFIG_ERROR;
    if (!(cutoff_scale > 0.0) || !isfinite(cutoff_scale))
        return PPFO_CONFIG_ERROR;
    if (!(beta >= 0.0) || !isfinite(beta))
        return PPFO_CONFIG_ERROR;
    const size_t length = n_channels * n_taps;
    double* w = (double*)malloc(length * sizeof(double));
    if (!w)
        return PPFO_CONFIG_ERROR;
    int st = ppfo_kaiser_window(length, beta, w);
    if (st != PPFO_OK) {
        free(w);
        return st;
    }
    const double step = M_PI * cutoff_scale / (2.0 * (double)n_channels);
    double sum = 0.0;
    for (size_t k = 0; k < length; ++k) {
        const double num = (double)(2 * (int64_t)k - (int64_t)(length - 1));
        const double v = ppfo_sinc(num * step) * w[k];
        out[k] = v;
        sum += v;
    }
    free(w);
    if (!isfinite(sum) || sum == 0.0)
        return PPFO_DEGENERATE_FILTER;
    for (size_t k = 0; k < length; ++k)
        out[k] /= sum;
    return PPFO_OK;
}

/* ---------------------------------------------------------------- flops */

/* include/ppf/fir.hpp:49-52 */
uint64_t ppfo_flops_for_fir(size_t n_channels, size_t n_taps, size_t n_spectra_out) {
    return (uint64_t)n_spectra_out * n_channels * n_taps * 4u;
}

static int is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }

static unsigned log2_exact(size_t n) {
    unsigned l = 0;
    while (((size_t)1 << l) < n)
        ++l;
    return l;
}

/* include/ppf/dft.hpp:28-35 */
uint64_t ppfo_flops_for_dft(size_t n_channels, size_t n_spectra) {
    const uint64_t n = n_channels;
    if (is_pow2(n_channels))
        return (uint64_t)n_spectra * 5u * n * log2_exact(n_channels);
    return (uint64_t)n_spectra * 8u * n * n;
}

/* ---------------------------------------------------------------- FIR */

/* include/ppf/fir.hpp:56-65 */
static int check_fir(size_t n_spectra_in, size_t n_channels, size_t n_taps) {
    if (n_channels == 0 || n_spectra_in == 0)
        return PPFO_CONFIG_ERROR;
    if (n_taps == 0)
        return PPFO_CONFIG_ERROR;
    if (n_spectra_in < n_taps)
        return PPFO_INSUFFICIENT_HISTORY;
    return PPFO_OK;
}

/* include/ppf/fir.hpp:158-212 with the per-element op sequence of
 * accumulate_spectrum (fir.hpp:85-110): product at t = 0, then one double
 * fma per tap in ascending t, round to f32. Taps quantized to f32 first
 * (quantize_taps, fir.hpp:69-74). With reference_order the t = 0 step is
 * fma(w, x, 0.0) as in ppf_fir_reference (fir.hpp:138-145). */
int ppfo_fir(const float* in, size_t n_spectra_in, size_t n_channels, size_t n_taps,
             const double* coeff_values, float* out, int reference_order) {
    int st = check_fir(n_spectra_in, n_channels, n_taps);
    if (st != PPFO_OK)
        return st;
    const size_t n_out = n_spectra_in - n_taps + 1;
    const size_t width = 2 * n_channels;
    float* taps = (float*)malloc(n_taps * n_channels * sizeof(float));
    if (!taps)
        return PPFO_CONFIG_ERROR;
    for (size_t k = 0; k < n_taps * n_channels; ++k)
        taps[k] = (float)coeff_values[k];
    for (size_t s = 0; s < n_out; ++s) {
        for (size_t e = 0; e < width; ++e) {
            const size_t c = e >> 1;
            const double w0 = (double)taps[c];
            const double x0 = (double)in[s * width + e];
            double acc = reference_order ? fma(w0, x0, 0.0) : w0 * x0;
            for (size_t t = 1; t < n_taps; ++t)
                acc = fma((double)taps[t * n_channels + c], (double)in[(s + t) * width + e], acc);
            out[s * width + e] = (float)acc;
        }
    }
    free(taps);
    return PPFO_OK;
}

/* ---------------------------------------------------------------- DFT */

/* include/ppf/dft.hpp:39-66: roots in double indexed by (k*m) mod N. */
int ppfo_dft_naive(const float* in, size_t n, float* out) {
    if (n == 0)
        return PPFO_CONFIG_ERROR;
    double* rr = (double*)malloc(n * sizeof(double));
    double* ri = (double*)malloc(n * sizeof(double));
    if (!rr || !ri) {
        free(rr);
        free(ri);
        return PPFO_CONFIG_ERROR;
    }
    for (size_t j = 0; j < n; ++j) {
        const double angle = -2.0 * M_PI * (double)j / (double)n;
        rr[j] = cos(angle);
        ri[j] = sin(angle);
    }
    for (size_t k = 0; k < n; ++k) {
        double acc_re = 0.0, acc_im = 0.0;
        for (size_t m = 0; m < n; ++m) {
            const size_t idx = (k * m) % n;
            const double xr = in[2 * m], xi = in[2 * m + 1];
            /* [contract] acc_re += xr*wr - xi*wi; acc_im += xr*wi + xi*wr
             * (dft.hpp:60-61) -> the first product fused into an fma */
            acc_re += fma(xr, rr[idx], -(xi * ri[idx]));
            acc_im += fma(xr, ri[idx], xi * rr[idx]);
        }
        out[2 * k] = (float)acc_re;
        out[2 * k + 1] = (float)acc_im;
    }
    free(rr);
    free(ri);
    return PPFO_OK;
}

/* include/ppf/dft.hpp:74-99 — bit reversal + per-stage f32 twiddles. */
typedef struct {
    size_t n;
    unsigned log2n;
    size_t* bitrev;
    float* tw_re; /* stage with half h stores its h roots at [h-1, 2h-2] */
    float* tw_im;
} fft_plan;

static int fft_plan_init(fft_plan* p, size_t n) {
    memset(p, 0, sizeof(*p));
    if (!is_pow2(n))
        return PPFO_UNSUPPORTED_SIZE;
    p->n = n;
    p->log2n = log2_exact(n);
    p->bitrev = (size_t*)malloc(n * sizeof(size_t));
    p->tw_re = (float*)malloc((n > 1 ? n - 1 : 1) * sizeof(float));
    p->tw_im = (float*)malloc((n > 1 ? n - 1 : 1) * sizeof(float));
    if (!p->bitrev || !p->tw_re || !p->tw_im)
        return PPFO_CONFIG_ERROR;
    for (size_t i = 0; i < n; ++i) {
        size_t r = 0;
        for (unsigned b = 0; b < p->log2n; ++b)
            r |= ((i >> b) & 1u) << (p->log2n - 1 - b);
        p->bitrev[i] = r;
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2;
        for (size_t j = 0; j < half; ++j) {
            const double angle = -2.0 * M_PI * (double)j / (double)len;
            p->tw_re[half - 1 + j] = (float)cos(angle);
            p->tw_im[half - 1 + j] = (float)sin(angle);
        }
    }
    return PPFO_OK;
}

static void fft_plan_free(fft_plan* p) {
    free(p->bitrev);
    free(p->tw_re);
    free(p->tw_im);
}

/* include/ppf/dft.hpp:105-134 (transform_planes) via 138-148 (transform) */
static void fft_transform(const fft_plan* p, float* row, float* re, float* im) {
    const size_t n = p->n;
    for (size_t i = 0; i < n; ++i) {
        re[i] = row[2 * i];
        im[i] = row[2 * i + 1];
    }
    for (size_t i = 0; i < n; ++i) {
        const size_t r = p->bitrev[i];
        if (i < r) {
            float t = re[i];
            re[i] = re[r];
            re[r] = t;
            t = im[i];
            im[i] = im[r];
            im[r] = t;
        }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2;
        const float* wr = p->tw_re + (half - 1);
        const float* wi = p->tw_im + (half - 1);
        for (size_t base = 0; base < n; base += len) {
            float* lo_re = re + base;
            float* lo_im = im + base;
            float* hi_re = lo_re + half;
            float* hi_im = lo_im + half;
            for (size_t j = 0; j < half; ++j) {
                const float br = hi_re[j];
                const float bi = hi_im[j];
                const float tr = fmaf(br, wr[j], -(bi * wi[j]));
                const float ti = fmaf(br, wi[j], bi * wr[j]);
                hi_re[j] = lo_re[j] - tr;
                hi_im[j] = lo_im[j] - ti;
                lo_re[j] += tr;
                lo_im[j] += ti;
            }
        }
    }
    for (size_t i = 0; i < n; ++i) {
        row[2 * i] = re[i];
        row[2 * i + 1] = im[i];
    }
}

/* include/ppf/dft.hpp:160-169 */
int ppfo_fft(float* row, size_t n) {
    if (n == 0)
        return PPFO_CONFIG_ERROR;
    fft_plan p;
    int st = fft_plan_init(&p, n);
    if (st != PPFO_OK) {
        fft_plan_free(&p);
        return st;
    }
    float* scratch = (float*)malloc(2 * n * sizeof(float));
    fft_transform(&p, row, scratch, scratch + n);
    free(scratch);
    fft_plan_free(&p);
    return PPFO_OK;
}

/* include/ppf/dft.hpp:175-235 (row-parallelism is irrelevant to results:
 * dft.hpp:171-174) */
int ppfo_channelize(const float* filtered, size_t n_rows, size_t n_channels, int fft_fallback,
                    float* out) {
    if (n_channels == 0)
        return PPFO_CONFIG_ERROR;
    if (n_rows == 0)
        return PPFO_OK;
    const int pow2 = is_pow2(n_channels);
    if (!pow2 && !fft_fallback)
        return PPFO_UNSUPPORTED_SIZE;
    const size_t n = n_channels;
    if (pow2) {
        fft_plan p;
        int st = fft_plan_init(&p, n);
        if (st != PPFO_OK) {
            fft_plan_free(&p);
            return st;
        }
        float* scratch = (float*)malloc(2 * n * sizeof(float));
        for (size_t s = 0; s < n_rows; ++s) {
            memcpy(out + 2 * s * n, filtered + 2 * s * n, 2 * n * sizeof(float));
            fft_transform(&p, out + 2 * s * n, scratch, scratch + n);
        }
        free(scratch);
        fft_plan_free(&p);
    } else {
        for (size_t s = 0; s < n_rows; ++s)
            ppfo_dft_naive(filtered + 2 * s * n, n, out + 2 * s * n);
    }
    return PPFO_OK;
}

int ppfo_fir_fft(const float* in, size_t n_spectra_in, size_t n_channels, size_t n_taps,
                 const double* coeff_values, int fft_fallback, float* out) {
    int st = check_fir(n_spectra_in, n_channels, n_taps);
    if (st != PPFO_OK)
        return st;
    if (!is_pow2(n_channels) && !fft_fallback)
        return PPFO_UNSUPPORTED_SIZE;
    const size_t n_out = n_spectra_in - n_taps + 1;
    float* filt = (float*)malloc(n_out * n_channels * 2 * sizeof(float));
    if (!filt)
        return PPFO_CONFIG_ERROR;
    st = ppfo_fir(in, n_spectra_in, n_channels, n_taps, coeff_values, filt, 0);
    if (st == PPFO_OK)
        st = ppfo_channelize(filt, n_out, n_channels, fft_fallback, out);
    free(filt);
    return st;
}

/* ---------------------------------------------------------------- stream */

/* include/ppf/pipeline.hpp:89-200 with carry_history (pipeline.hpp:55-73)
 * and process_block (pipeline.hpp:121-136), reading an in-memory source in
 * requests of block_spectra*C*8 bytes (istringstream read/gcount/eof). */
int ppfo_process_stream(size_t n_channels, size_t n_taps, size_t block_spectra, int fft_fallback,
                        int zero_prime, const double* coeff_values, const uint8_t* src,
                        size_t src_len, uint8_t* out, ppfo_stream_state* state) {
    memset(state, 0, sizeof(*state));
    /* PpfConfig::validate, pipeline.hpp:28-38 */
    if (n_channels == 0 || n_taps == 0 || block_spectra < n_taps)
        return PPFO_CONFIG_ERROR;
    const size_t sample_bytes = 8;
    const size_t spectrum_bytes = n_channels * sample_bytes;
    const size_t io_size = block_spectra * spectrum_bytes;

    /* history: at most n_taps-1 spectra */
    float* history = (float*)calloc((n_taps > 1 ? n_taps - 1 : 1) * n_channels * 2, sizeof(float));
    size_t hist_spectra = 0;
    if (zero_prime)
        hist_spectra = n_taps - 1; /* pipeline.hpp:110-111 */

    /* sample carry never exceeds one read + one spectrum */
    const size_t carry_cap = io_size / sample_bytes + n_channels + 1;
    float* sample_carry = (float*)malloc(carry_cap * 2 * sizeof(float));
    size_t carry_n = 0;
    uint8_t byte_carry[8];
    size_t byte_carry_n = 0;
    uint64_t stream_offset = 0;
    size_t pos = 0;
    size_t out_pos = 0;

    float* joined = (float*)malloc((block_spectra + n_taps + 1) * n_channels * 2 * sizeof(float));
    float* filt = (float*)malloc((block_spectra + n_taps + 1) * n_channels * 2 * sizeof(float));
    int st = PPFO_OK;

    for (;;) {
        const size_t got = (src_len - pos) < io_size ? (src_len - pos) : io_size;
        const int eof = got < io_size;
        if (got == 0)
            break;
        const uint8_t* data = src + pos;
        size_t avail = got;
        pos += got;

        if (byte_carry_n != 0) { /* pipeline.hpp:151-163 */
            const size_t need = sample_bytes - byte_carry_n;
            const size_t take = need < avail ? need : avail;
            memcpy(byte_carry + byte_carry_n, data, take);
            byte_carry_n += take;
            data += take;
            avail -= take;
            if (byte_carry_n == sample_bytes) {
                memcpy(sample_carry + 2 * carry_n, byte_carry, sample_bytes);
                ++carry_n;
                byte_carry_n = 0;
            }
        }
        const size_t full_samples = avail / sample_bytes;
        const size_t tail = avail % sample_bytes;
        memcpy(sample_carry + 2 * carry_n, data, full_samples * sample_bytes);
        carry_n += full_samples;
        if (tail != 0) {
            memcpy(byte_carry, data + full_samples * sample_bytes, tail);
            byte_carry_n = tail;
        }
        stream_offset += got;

        const size_t full_spectra = carry_n / n_channels;
        if (full_spectra != 0) { /* pipeline.hpp:174-184 */
            const size_t block_n = full_spectra * n_channels;
            state->bytes_in += full_spectra * spectrum_bytes;
            /* carry_history: joined = history ++ block */
            memcpy(joined, history, hist_spectra * n_channels * 2 * sizeof(float));
            memcpy(joined + hist_spectra * n_channels * 2, sample_carry, block_n * 2 * sizeof(float));
            const size_t joined_spectra = hist_spectra + full_spectra;
            const size_t keep = (n_taps - 1) < joined_spectra ? (n_taps - 1) : joined_spectra;
            memcpy(history, joined + (joined_spectra - keep) * n_channels * 2,
                   keep * n_channels * 2 * sizeof(float));
            hist_spectra = keep;
            memmove(sample_carry, sample_carry + 2 * block_n, (carry_n - block_n) * 2 * sizeof(float));
            carry_n -= block_n;
            if (joined_spectra >= n_taps) { /* process_block, pipeline.hpp:121-136 */
                const size_t n_out = joined_spectra - n_taps + 1;
                st = ppfo_fir(joined, joined_spectra, n_channels, n_taps, coeff_values, filt, 0);
                if (st == PPFO_OK)
                    st = ppfo_channelize(filt, n_out, n_channels, fft_fallback,
                                         (float*)(out + out_pos));
                if (st != PPFO_OK)
                    goto done;
                out_pos += n_out * spectrum_bytes;
                state->spectra_processed += n_out;
                state->bytes_out += n_out * spectrum_bytes;
            }
        }
        if (eof)
            break;
    }
    if (byte_carry_n != 0) { /* pipeline.hpp:190-192 */
        state->error_offset = stream_offset - byte_carry_n;
        st = PPFO_DECODE_ERROR;
        goto done;
    }
    state->dropped_samples += carry_n; /* pipeline.hpp:194 */
done:
    free(history);
    free(sample_carry);
    free(joined);
    free(filt);
    return st;
}

/* cli.hpp:307-317. The product (double)re*re is exact (24-bit mantissas), so
 * whether a compiler contracts re*re + im*im into an fma does not change p. */
int ppfo_mean_power(const float* bins, size_t n_spectra, size_t n_channels, double* mean) {
    if (n_channels == 0)
        return PPFO_CONFIG_ERROR;
    for (size_t c = 0; c < n_channels; ++c)
        mean[c] = 0.0;
    for (size_t s = 0; s < n_spectra; ++s) {
        for (size_t c = 0; c < n_channels; ++c) {
            const double re = (double)bins[2 * (s * n_channels + c)];
            const double im = (double)bins[2 * (s * n_channels + c) + 1];
            mean[c] += re * re + im * im;
        }
    }
    if (n_spectra != 0)
        for (size_t c = 0; c < n_channels; ++c)
            mean[c] /= (double)n_spectra;
    return PPFO_OK;
}

/* ---- synthetic workload (bench input; bytes identical to ppfg_synth) ---------- */
static uint64_t synth_splitmix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

static int synth_irwin_hall4(uint64_t z) {
    return (int)((z & 0xffff) + ((z >> 16) & 0xffff) + ((z >> 32) & 0xffff) + (z >> 48)) - 131070;
}

int ppfo_synth(size_t n_channels, uint64_t seed, uint64_t first_sample, size_t n_samples,
               float* out) {
    if (n_channels == 0)
        return PPFO_CONFIG_ERROR;
    const uint64_t M = 10 * (uint64_t)n_channels, f10 = (10 * (uint64_t)n_channels) / 8 + 3;
    float* tone = (float*)malloc(sizeof(float) * 2 * M);
    if (!tone)
        return PPFO_OTHER;
    for (uint64_t k = 0; k < M; ++k) {
        const double a = 2.0 * M_PI * (double)k / (double)M;
        tone[2 * k] = (float)cos(a);
        tone[2 * k + 1] = (float)sin(a);
    }
    const uint64_t golden = 0x9e3779b97f4a7c15ULL;
    const float scale = 2.64293e-05f;
    for (size_t i = 0; i < n_samples; ++i) {
        const uint64_t n = first_sample + i;
        const uint64_t t = (f10 * n) % M;
        const float gr = (float)synth_irwin_hall4(synth_splitmix64(seed + (2 * n + 1) * golden)) * scale;
        const float gi = (float)synth_irwin_hall4(synth_splitmix64(seed + (2 * n + 2) * golden)) * scale;
        out[2 * i] = tone[2 * t] + gr;
        out[2 * i + 1] = tone[2 * t + 1] + gi;
    }
    free(tone);
    return PPFO_OK;
}
