// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/ppf/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libppfref*.so. TEST INFRASTRUCTURE ONLY: used by tests/ to pin
// the C restatement (oracle/ppf_oracle.c) and the golden vectors, and by
// bench.py --impl reference / cpu_baseline to time the reference's own CPU
// path. No reference source is copied; this file only calls its public API.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "ppf/bench.hpp"
#include "ppf/coeff.hpp"
#include "ppf/dft.hpp"
#include "ppf/errors.hpp"
#include "ppf/fir.hpp"
#include "ppf/pipeline.hpp"

namespace {

thread_local std::string g_err;
thread_local std::uint64_t g_offset = 0;

// same numbering as include/ppfg.h
int map_exception() {
    try {
        throw;
    } catch (const ppf::insufficient_history_error& e) {
        g_err = e.what();
        return 2;
    } catch (const ppf::unsupported_size_error& e) {
        g_err = e.what();
        return 3;
    } catch (const ppf::config_error& e) {
        g_err = e.what();
        return 1;
    } catch (const ppf::degenerate_filter_error& e) {
        g_err = e.what();
        return 4;
    } catch (const ppf::decode_error& e) {
        g_err = e.what();
        g_offset = e.byte_offset;
        return 5;
    } catch (const ppf::io_error& e) {
        g_err = e.what();
        return 6;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 9;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

ppf::FilterCoefficients make_coeffs(std::size_t nc, std::size_t nt, const double* v) {
    ppf::FilterCoefficients c;
    c.n_channels = nc;
    c.n_taps = nt;
    c.values.assign(v, v + nc * nt);
    return c;
}

ppf::SampleBlock make_block(const float* in, std::size_t n_spectra, std::size_t nc) {
    ppf::SampleBlock b;
    b.n_channels = nc;
    b.samples.resize(n_spectra * nc);
    std::memcpy(b.samples.data(), in, n_spectra * nc * sizeof(ppf::ComplexSample));
    return b;
}

} // namespace

extern "C" {

const char* ppfr_last_error() { return g_err.c_str(); }
std::uint64_t ppfr_last_error_offset() { return g_offset; }

int ppfr_generate_prototype(std::size_t nc, std::size_t nt, double beta, int rectangular,
                            double* out) {
    try {
        const auto w = rectangular ? ppf::WindowSpec::rectangular() : ppf::WindowSpec::kaiser(beta);
        const auto c = ppf::generate_prototype(nc, nt, w);
        std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

double ppfr_bessel_i0(double x, int* status) {
    try {
        *status = 0;
        return ppf::bessel_i0(x);
    } catch (...) {
        *status = map_exception();
        return 0.0;
    }
}

// fir.hpp:123-151 (reference=1) or fir.hpp:158-212 (reference=0)
int ppfr_fir(const float* in, std::size_t n_spectra_in, std::size_t nc, std::size_t nt,
             const double* coeffs, float* out, int reference, unsigned workers) {
    try {
        const auto block = make_block(in, n_spectra_in, nc);
        const auto c = make_coeffs(nc, nt, coeffs);
        const ppf::FilteredBlock f =
            reference ? ppf::ppf_fir_reference(block, c) : ppf::ppf_fir_optimized(block, c, workers);
        std::memcpy(out, f.spectra.data(), f.spectra.size() * sizeof(ppf::ComplexSample));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ppfr_dft_naive(const float* in, std::size_t n, float* out) {
    try {
        const auto* p = reinterpret_cast<const ppf::ComplexSample*>(in);
        const auto r = ppf::dft_naive(std::span<const ppf::ComplexSample>(p, n));
        std::memcpy(out, r.data(), n * sizeof(ppf::ComplexSample));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ppfr_fft(const float* in, std::size_t n, float* out) {
    try {
        const auto* p = reinterpret_cast<const ppf::ComplexSample*>(in);
        const auto r = ppf::fft(std::span<const ppf::ComplexSample>(p, n));
        std::memcpy(out, r.data(), n * sizeof(ppf::ComplexSample));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

int ppfr_channelize(const float* in, std::size_t rows, std::size_t nc, int fft_fallback,
                    unsigned workers, float* out) {
    try {
        ppf::FilteredBlock f;
        f.n_channels = nc;
        f.n_spectra_out = rows;
        f.spectra.resize(rows * nc);
        std::memcpy(f.spectra.data(), in, rows * nc * sizeof(ppf::ComplexSample));
        const auto o = ppf::channelize_block(f, fft_fallback != 0, workers);
        std::memcpy(out, o.bins.data(), o.bins.size() * sizeof(ppf::ComplexSample));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// the library one-shot used by the reference tests (pipeline_test.cpp:40-51):
// ppf_fir_optimized then channelize_block
int ppfr_fir_fft(const float* in, std::size_t n_spectra_in, std::size_t nc, std::size_t nt,
                 const double* coeffs, int fft_fallback, unsigned workers, float* out) {
    try {
        const auto block = make_block(in, n_spectra_in, nc);
        const auto c = make_coeffs(nc, nt, coeffs);
        const auto f = ppf::ppf_fir_optimized(block, c, workers);
        const auto o = ppf::channelize_block(f, fft_fallback != 0, workers);
        std::memcpy(out, o.bins.data(), o.bins.size() * sizeof(ppf::ComplexSample));
        return 0;
    } catch (...) {
        return map_exception();
    }
}

struct ppfr_stream_state {
    std::uint64_t spectra_processed, bytes_in, bytes_out, dropped_samples, error_offset;
};

// pipeline.hpp:89-200 over an in-memory source / sink
int ppfr_process_stream(std::size_t nc, std::size_t nt, std::size_t block_spectra,
                        int fft_fallback, int zero_prime, const double* coeffs,
                        const std::uint8_t* src, std::size_t src_len, std::uint8_t* out,
                        std::size_t* out_len, unsigned workers, ppfr_stream_state* st) {
    try {
        ppf::PpfConfig cfg;
        cfg.n_channels = nc;
        cfg.n_taps = nt;
        cfg.block_spectra = block_spectra;
        cfg.fft_fallback = fft_fallback != 0;
        ppf::StreamOptions opt;
        opt.workers = workers;
        opt.zero_prime = zero_prime != 0;
        ppf::FilterCoefficients c;
        if (coeffs) {
            c = make_coeffs(nc, nt, coeffs);
            opt.coefficients = &c;
        }
        std::istringstream source(std::string(reinterpret_cast<const char*>(src), src_len));
        std::ostringstream sink;
        const auto s = ppf::process_stream(cfg, source, sink, opt);
        const std::string bytes = sink.str();
        std::memcpy(out, bytes.data(), bytes.size());
        *out_len = bytes.size();
        st->spectra_processed = s.spectra_processed;
        st->bytes_in = s.bytes_in;
        st->bytes_out = s.bytes_out;
        st->dropped_samples = s.dropped_samples;
        st->error_offset = 0;
        return 0;
    } catch (...) {
        const int rc = map_exception();
        st->error_offset = g_offset;
        return rc;
    }
}

// The reference's own compute pass (bench.hpp:129-150): block-partitioned
// carry_history -> ppf_fir_optimized -> channelize_block over a resident
// input, `reps` times. Returns the wall seconds of each rep in secs[].
// Input is the caller's (so the CPU arm can time the same bytes as the GPU).
int ppfr_compute_pass(const float* in, std::size_t total_spectra, std::size_t nc, std::size_t nt,
                      const double* coeffs, std::size_t block_spectra, unsigned workers,
                      unsigned reps, double* secs, std::uint64_t* emitted_out) {
    try {
        const auto c = make_coeffs(nc, nt, coeffs);
        const auto* samples = reinterpret_cast<const ppf::ComplexSample*>(in);
        for (unsigned r = 0; r < reps; ++r) {
            const double t0 = ppf::detail::steady_seconds();
            ppf::StreamState state;
            ppf::SampleBlock block;
            block.n_channels = nc;
            std::uint64_t emitted = 0;
            for (std::size_t s = 0; s < total_spectra; s += block_spectra) {
                const std::size_t n = std::min(block_spectra, total_spectra - s);
                block.samples.assign(samples + s * nc, samples + (s + n) * nc);
                const ppf::SampleBlock joined = ppf::carry_history(state, block, nt);
                if (joined.n_spectra() < nt)
                    continue;
                const auto filtered = ppf::ppf_fir_optimized(joined, c, workers);
                const auto chan = ppf::channelize_block(filtered, true, workers);
                emitted += chan.n_spectra;
            }
            secs[r] = ppf::detail::steady_seconds() - t0;
            *emitted_out = emitted;
        }
        return 0;
    } catch (...) {
        return map_exception();
    }
}

// bench.hpp:97-208 as-is (includes its scratch-file end-to-end pass)
int ppfr_run_benchmark(std::size_t nc, std::size_t nt, std::size_t total_spectra,
                       unsigned workers, unsigned reps, double* m_c, double* m_b,
                       double* wall_compute, double* bandwidth) {
    try {
        ppf::PpfConfig cfg;
        cfg.n_channels = nc;
        cfg.n_taps = nt;
        ppf::BenchOptions opt;
        opt.repetitions = reps;
        const auto r = ppf::run_benchmark(cfg, total_spectra, workers, opt);
        *m_c = r.m_c;
        *m_b = r.m_b;
        *wall_compute = r.wall_compute_sec;
        *bandwidth = r.bandwidth_gb_per_sec;
        return 0;
    } catch (...) {
        return map_exception();
    }
}

} // extern "C"
