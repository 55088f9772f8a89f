// ppf_gpu/ppf.hpp — C++ drop-in for the reference's public PPF API
// (/root/reference/proj/include/ppf/*.hpp) on top of libppfg.so's C-ABI
// (include/ppfg.h). Same type names, fields, function signatures and
// exception classes; the FIR, FFT, fused FIR+FFT and streaming bodies run on
// the B200 (sm_100a) kernels behind the C-ABI.
//
// Namespace: ppf_gpu by default. Define PPF_GPU_NS=ppf before including (the
// shims in include/ppf_dropin/ppf/*.hpp do) to compile reference callers
// unchanged: they switch by include path + linking -lppfg.
//
// Results: ppf_fir_optimized / ppf_fir_reference / channelize_block / fft /
// dft_naive / process_stream are bit-identical to the reference (FP64 FIR in
// the reference's operation order, the reference's radix-2 butterflies and
// twiddles). `workers` arguments are accepted for signature compatibility;
// work is partitioned over CUDA threads and never changes a result
// (SPEC.md:141,163). The device is the calling thread's current CUDA device.
#pragma once

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <functional>
#include <istream>
#include <list>
#include <mutex>
#include <numbers>
#include <optional>
#include <ostream>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <sys/mman.h>
#include <utility>
#include <vector>

#include "ppfg.h"

#ifndef PPF_GPU_NS
#define PPF_GPU_NS ppf_gpu
#endif

namespace PPF_GPU_NS {

// ============================================================ errors.hpp
struct config_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct insufficient_history_error : config_error {
    using config_error::config_error;
};
struct unsupported_size_error : config_error {
    using config_error::config_error;
};
struct degenerate_filter_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct decode_error : std::runtime_error {
    decode_error(const std::string& what, std::size_t offset)
        : std::runtime_error(what + " at byte offset " + std::to_string(offset)),
          byte_offset(offset) {}
    std::size_t byte_offset;
};
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// device-side failures have no reference counterpart
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
// ppfg_status -> the reference's exception classes (include/ppfg.h)
[[noreturn]] inline void raise(int status) {
    const std::string msg = ppfg_last_error();
    switch (status) {
    case PPFG_CONFIG_ERROR:
        throw config_error(msg);
    case PPFG_INSUFFICIENT_HISTORY:
        throw insufficient_history_error(msg);
    case PPFG_UNSUPPORTED_SIZE:
        throw unsupported_size_error(msg);
    case PPFG_DEGENERATE_FILTER:
        throw degenerate_filter_error(msg);
    case PPFG_DECODE_ERROR: {
        // the C-ABI message already carries "at byte offset N"
        const auto off = static_cast<std::size_t>(ppfg_last_error_offset());
        const std::string tail = " at byte offset " + std::to_string(off);
        std::string base = msg;
        if (base.size() >= tail.size() && base.compare(base.size() - tail.size(), tail.size(), tail) == 0)
            base.resize(base.size() - tail.size());
        throw decode_error(base, off);
    }
    case PPFG_IO_ERROR:
        throw io_error(msg);
    case PPFG_DOMAIN_ERROR:
        throw std::domain_error(msg);
    default:
        throw device_error(msg);
    }
}
inline void check(int status) {
    if (status != PPFG_OK)
        raise(status);
}
} // namespace detail

// ============================================================ coeff.hpp
inline constexpr double kDefaultKaiserBeta = 9.0;
inline constexpr double kDefaultCutoffScale = 1.5;
inline constexpr double kBesselMaxArg = 700.0;

struct WindowSpec {
    enum class Kind { kaiser, rectangular };
    Kind kind = Kind::kaiser;
    double beta = kDefaultKaiserBeta;
    static WindowSpec kaiser(double b) { return {Kind::kaiser, b}; }
    static WindowSpec rectangular() { return {Kind::rectangular, 0.0}; }
    double effective_beta() const { return kind == Kind::rectangular ? 0.0 : beta; }
    void validate() const {
        if (!(beta >= 0.0) || !std::isfinite(beta))
            throw config_error("window beta must be finite and >= 0");
    }
};

struct FilterCoefficients {
    std::size_t n_channels = 0;
    std::size_t n_taps = 0;
    std::vector<double> values; // tap-major: values[t * n_channels + c]
    double at(std::size_t tap, std::size_t channel) const {
        return values[tap * n_channels + channel];
    }
};

inline double sinc(double x) { return x == 0.0 ? 1.0 : std::sin(x) / x; }

inline double bessel_i0(double x) {
    if (!(std::fabs(x) <= kBesselMaxArg))
        throw std::domain_error("bessel_i0: |x| must be <= 700");
    const double q = 0.25 * x * x;
    double term = 1.0, total = 1.0;
    for (int k = 1; k < 10000; ++k) {
        term *= q / (static_cast<double>(k) * static_cast<double>(k));
        total += term;
        if (term < total * 1e-17)
            break;
    }
    return total;
}

inline std::vector<double> kaiser_window(std::size_t length, double beta) {
    if (length == 0)
        throw config_error("kaiser_window: length must be >= 1");
    if (!(beta >= 0.0) || !std::isfinite(beta))
        throw config_error("kaiser_window: beta must be finite and >= 0");
    std::vector<double> w(length, 1.0);
    if (length == 1 || beta == 0.0)
        return w;
    const double norm = bessel_i0(beta);
    const double span = static_cast<double>(length - 1);
    for (std::size_t k = 0; k < length; ++k) {
        const double r =
            static_cast<double>(2 * static_cast<std::int64_t>(k) - static_cast<std::int64_t>(length - 1)) /
            span;
        w[k] = bessel_i0(beta * std::sqrt(std::fma(-r, r, 1.0))) / norm;
    }
    return w;
}

// coeff.hpp:110-144, computed by libppfg (bit-identical to the reference)
inline FilterCoefficients generate_prototype(std::size_t n_channels, std::size_t n_taps,
                                             WindowSpec window,
                                             double cutoff_scale = kDefaultCutoffScale) {
    if (n_channels == 0 || n_taps == 0)
        throw config_error("generate_prototype: n_channels and n_taps must be >= 1");
    window.validate();
    FilterCoefficients c;
    c.n_channels = n_channels;
    c.n_taps = n_taps;
    c.values.resize(n_channels * n_taps);
    detail::check(ppfg_generate_prototype(n_channels, n_taps, window.effective_beta(),
                                          cutoff_scale, c.values.data()));
    return c;
}

// PPFC v1 coefficient files (coeff.hpp:146-229 layout)
inline constexpr char kCoeffMagic[4] = {'P', 'P', 'F', 'C'};
inline constexpr std::uint32_t kCoeffFormatVersion = 1;

struct CoefficientFile {
    FilterCoefficients coeffs;
    double beta = 0.0;
};

inline void write_coefficients(std::ostream& os, const FilterCoefficients& coeffs, double beta) {
    auto put = [&](const void* p, std::size_t n) { os.write(static_cast<const char*>(p), n); };
    put(kCoeffMagic, 4);
    const std::uint32_t hdr[3] = {kCoeffFormatVersion, static_cast<std::uint32_t>(coeffs.n_channels),
                                  static_cast<std::uint32_t>(coeffs.n_taps)};
    put(hdr, sizeof hdr);
    put(&beta, sizeof beta);
    for (double v : coeffs.values) {
        const float f = static_cast<float>(v);
        put(&f, sizeof f);
    }
    if (!os)
        throw io_error("write_coefficients: write failed");
}

inline void write_coefficients_text(std::ostream& os, const FilterCoefficients& coeffs) {
    for (double v : coeffs.values) {
        char line[64];
        std::snprintf(line, sizeof line, "%.9g\n", static_cast<double>(static_cast<float>(v)));
        os << line;
    }
    if (!os)
        throw io_error("write_coefficients_text: write failed");
}

inline CoefficientFile read_coefficients(std::istream& is) {
    auto get = [&](void* p, std::size_t n) {
        is.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
        return is.gcount() == static_cast<std::streamsize>(n);
    };
    char magic[4] = {};
    if (!get(magic, 4) || std::memcmp(magic, kCoeffMagic, 4) != 0)
        throw decode_error("read_coefficients: bad magic", 0);
    std::uint32_t version = 0, nc = 0, nt = 0;
    double beta = 0.0;
    if (!get(&version, 4) || version != kCoeffFormatVersion)
        throw decode_error("read_coefficients: unsupported format version", 4);
    if (!get(&nc, 4) || !get(&nt, 4) || !get(&beta, 8))
        throw decode_error("read_coefficients: truncated header", 8);
    if (nc == 0 || nt == 0)
        throw decode_error("read_coefficients: zero channel or tap count", 8);
    CoefficientFile f;
    f.beta = beta;
    f.coeffs.n_channels = nc;
    f.coeffs.n_taps = nt;
    f.coeffs.values.resize(static_cast<std::size_t>(nc) * nt);
    for (std::size_t k = 0; k < f.coeffs.values.size(); ++k) {
        float v = 0.0f;
        if (!get(&v, 4))
            throw decode_error("read_coefficients: truncated values", 20 + k * 4);
        f.coeffs.values[k] = v;
    }
    return f;
}

// ============================================================ fir.hpp
using ComplexSample = std::complex<float>;

struct SampleBlock {
    std::vector<ComplexSample> samples;
    std::size_t n_channels = 0;
    std::size_t n_spectra() const { return n_channels ? samples.size() / n_channels : 0; }
    void validate() const {
        if (n_channels == 0)
            throw config_error("SampleBlock: n_channels must be >= 1");
        if (samples.empty() || samples.size() % n_channels != 0)
            throw config_error("SampleBlock: sample count must be a positive multiple of n_channels");
    }
};

struct FilteredBlock {
    std::vector<ComplexSample> spectra;
    std::size_t n_channels = 0;
    std::size_t n_spectra_out = 0;
};

inline std::uint64_t flops_for_fir(std::size_t n_channels, std::size_t n_taps,
                                   std::size_t n_spectra_out) {
    return ppfg_flops_for_fir(n_channels, n_taps, n_spectra_out);
}

// A device plan owned by a C++ value (RAII over ppfg_plan).
class Plan {
public:
    Plan() = default;
    Plan(std::size_t n_channels, std::size_t n_taps, const double* values, std::uint32_t flags = PPFG_EXACT,
         int device = -1) {
        detail::check(ppfg_plan_create(&h_, n_channels, n_taps, values, flags, device));
    }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    Plan(Plan&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Plan& operator=(Plan&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    ~Plan() { ppfg_plan_destroy(h_); }
    ppfg_plan get() const { return h_; }

private:
    ppfg_plan h_ = nullptr;
};

namespace detail {
// Large result vectors are freshly allocated on every call (the reference API
// returns them by value); above glibc's mmap threshold each call page-faults
// them in 4 KB at a time. Ask for transparent huge pages on the vector's
// storage before its first touch (a hint: no effect where THP is disabled).
template <class T>
inline void reserve_huge(std::vector<T>& v, std::size_t n) {
    v.reserve(n);
    constexpr std::uintptr_t kHuge = std::uintptr_t(2) << 20;
    const std::size_t bytes = n * sizeof(T);
    if (bytes < 2 * kHuge)
        return;
    const std::uintptr_t b = reinterpret_cast<std::uintptr_t>(v.data());
    const std::uintptr_t lo = (b + kHuge - 1) & ~(kHuge - 1), hi = (b + bytes) & ~(kHuge - 1);
    if (hi > lo)
        ::madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
}

// Process-wide cache of device plans for the one-shot calls (ppf_fir_*,
// channelize_block): the reference API is stateless and a caller looping per
// block (bench.hpp:129-150, pipeline.hpp:121-136) would otherwise pay plan
// creation — tap / twiddle uploads, streams, events — and a fresh pinned
// staging area on every call. Plans are keyed by (device, C, T, flags,
// coefficient values); a plan is leased to one call at a time (plans are not
// thread-safe), concurrent callers get their own, and at most kMaxIdle idle
// plans are kept (least recently used dropped first).
class PlanCache {
public:
    struct Key {
        int device = 0;
        std::size_t n_channels = 0, n_taps = 0;
        std::uint32_t flags = 0;
        std::vector<double> values;
        bool operator==(const Key& o) const {
            return device == o.device && n_channels == o.n_channels && n_taps == o.n_taps &&
                   flags == o.flags && values == o.values;
        }
    };
    class Lease {
    public:
        Lease(PlanCache* c, Key k, ppfg_plan p) : c_(c), k_(std::move(k)), p_(p) {}
        Lease(const Lease&) = delete;
        Lease& operator=(const Lease&) = delete;
        ~Lease() { c_->give_back(std::move(k_), p_); }
        ppfg_plan get() const { return p_; }

    private:
        PlanCache* c_;
        Key k_;
        ppfg_plan p_;
    };
    static PlanCache& instance() {
        static PlanCache* c = new PlanCache(); // leaked on purpose: no exit-order issues
        return *c;
    }
    Lease acquire(std::size_t n_channels, std::size_t n_taps, const double* values,
                  std::uint32_t flags = PPFG_EXACT) {
        Key k;
        check(ppfg_current_device(&k.device));
        k.n_channels = n_channels;
        k.n_taps = n_taps;
        k.flags = flags;
        if (n_taps)
            k.values.assign(values, values + n_channels * n_taps);
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (auto it = idle_.begin(); it != idle_.end(); ++it) {
                if (it->first == k) {
                    ppfg_plan p = it->second;
                    idle_.erase(it);
                    return Lease(this, std::move(k), p);
                }
            }
        }
        ppfg_plan p = nullptr;
        check(ppfg_plan_create(&p, n_channels, n_taps, n_taps ? k.values.data() : nullptr, flags,
                               k.device));
        return Lease(this, std::move(k), p);
    }

private:
    static constexpr std::size_t kMaxIdle = 8;
    void give_back(Key k, ppfg_plan p) {
        std::lock_guard<std::mutex> lk(mu_);
        idle_.emplace_front(std::move(k), p);
        while (idle_.size() > kMaxIdle) {
            ppfg_plan_destroy(idle_.back().second);
            idle_.pop_back();
        }
    }
    std::mutex mu_;
    std::list<std::pair<Key, ppfg_plan>> idle_; // most recently used first
};

inline void check_fir_preconditions(const SampleBlock& input, const FilterCoefficients& coeffs) {
    input.validate();
    if (coeffs.n_channels == 0 || coeffs.n_taps == 0 ||
        coeffs.values.size() != coeffs.n_channels * coeffs.n_taps)
        throw config_error("fir: malformed coefficient set");
    if (input.n_channels != coeffs.n_channels)
        throw config_error("fir: input channel count does not match coefficients");
    if (input.n_spectra() < coeffs.n_taps)
        throw insufficient_history_error("fir: need at least n_taps input spectra");
}

inline FilteredBlock run_fir(const SampleBlock& input, const FilterCoefficients& coeffs,
                             bool reference_order) {
    check_fir_preconditions(input, coeffs);
    FilteredBlock out;
    out.n_channels = input.n_channels;
    out.n_spectra_out = input.n_spectra() - coeffs.n_taps + 1;
    detail::reserve_huge(out.spectra, out.n_spectra_out * out.n_channels);
    out.spectra.resize(out.n_spectra_out * out.n_channels);
    auto p = PlanCache::instance().acquire(coeffs.n_channels, coeffs.n_taps, coeffs.values.data());
    auto fn = reference_order ? ppfg_fir_reference_order : ppfg_fir;
    detail::check(fn(p.get(), input.samples.data(), input.n_spectra(), out.spectra.data(),
                     PPFG_MEM_HOST, nullptr));
    return out;
}
} // namespace detail

// fir.hpp:123-151
inline FilteredBlock ppf_fir_reference(const SampleBlock& input, const FilterCoefficients& coeffs) {
    return detail::run_fir(input, coeffs, true);
}

// fir.hpp:158-212
inline FilteredBlock ppf_fir_optimized(const SampleBlock& input, const FilterCoefficients& coeffs,
                                       unsigned workers) {
    if (workers == 0)
        throw config_error("fir: workers must be >= 1");
    return detail::run_fir(input, coeffs, false);
}

// ============================================================ dft.hpp
struct ChannelizedOutput {
    std::vector<ComplexSample> bins;
    std::size_t n_channels = 0;
    std::size_t n_spectra = 0;
};

inline bool is_power_of_two(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }

inline std::uint64_t flops_for_dft(std::size_t n_channels, std::size_t n_spectra) {
    return ppfg_flops_for_dft(n_channels, n_spectra);
}

inline std::vector<ComplexSample> dft_naive(std::span<const ComplexSample> spectrum) {
    if (spectrum.empty())
        throw config_error("dft_naive: empty spectrum");
    std::vector<ComplexSample> out(spectrum.size());
    detail::check(ppfg_dft_naive(spectrum.data(), spectrum.size(), out.data()));
    return out;
}

inline std::vector<ComplexSample> fft(std::span<const ComplexSample> spectrum) {
    if (spectrum.empty())
        throw config_error("fft: empty spectrum");
    std::vector<ComplexSample> out(spectrum.size());
    detail::check(ppfg_fft(spectrum.data(), spectrum.size(), out.data()));
    return out;
}

// dft.hpp:72-156: a reusable transform of a fixed power-of-two size, here a
// device plan; transform() runs one row (scratch is unused).
class FftPlan {
public:
    explicit FftPlan(std::size_t n) : n_(n) {
        if (!is_power_of_two(n))
            throw unsupported_size_error("fft: size must be a power of two");
        plan_ = Plan(n, 0, nullptr);
    }
    std::size_t size() const { return n_; }
    void transform(ComplexSample* a, float* /*scratch*/) const {
        detail::check(ppfg_channelize(plan_.get(), a, 1, a, 0, PPFG_MEM_HOST, nullptr));
    }

private:
    std::size_t n_;
    Plan plan_;
};

// dft.hpp:175-235
inline ChannelizedOutput channelize_block(const FilteredBlock& filtered, bool fft_fallback = true,
                                          unsigned workers = 1) {
    if (filtered.n_channels == 0)
        throw config_error("channelize_block: n_channels must be >= 1");
    if (filtered.spectra.size() != filtered.n_spectra_out * filtered.n_channels)
        throw config_error("channelize_block: malformed filtered block");
    if (workers == 0)
        throw config_error("channelize_block: workers must be >= 1");
    ChannelizedOutput out;
    out.n_channels = filtered.n_channels;
    out.n_spectra = filtered.n_spectra_out;
    if (out.n_spectra == 0)
        return out;
    if (!is_power_of_two(out.n_channels) && !fft_fallback)
        throw unsupported_size_error(
            "channelize_block: non-power-of-two channel count with fallback disabled");
    detail::reserve_huge(out.bins, filtered.spectra.size());
    out.bins.resize(filtered.spectra.size());
    auto p = detail::PlanCache::instance().acquire(filtered.n_channels, 0, nullptr);
    detail::check(ppfg_channelize(p.get(), filtered.spectra.data(), out.n_spectra, out.bins.data(),
                                  fft_fallback ? 1 : 0, PPFG_MEM_HOST, nullptr));
    return out;
}

// ============================================================ pipeline.hpp
inline constexpr std::size_t kDefaultBlockSpectra = 4096;
inline constexpr std::uint64_t kDefaultReferenceRate = 6'500'000'000ull;

struct PpfConfig {
    std::size_t n_channels = 0;
    std::size_t n_taps = 0;
    WindowSpec window;
    std::size_t block_spectra = kDefaultBlockSpectra;
    std::uint64_t reference_rate_bytes_per_sec = kDefaultReferenceRate;
    bool fft_fallback = true;
    void validate() const {
        if (n_channels == 0)
            throw config_error("config: n_channels must be >= 1");
        if (n_taps == 0)
            throw config_error("config: n_taps must be >= 1");
        if (block_spectra < n_taps)
            throw config_error("config: block_spectra must be >= n_taps");
        if (reference_rate_bytes_per_sec == 0)
            throw config_error("config: reference rate must be > 0");
        window.validate();
    }
};

struct StreamState {
    std::vector<ComplexSample> history;
    std::uint64_t spectra_processed = 0;
    std::uint64_t bytes_in = 0;
    std::uint64_t bytes_out = 0;
    std::uint64_t dropped_samples = 0;
};

// pipeline.hpp:55-73 (host bookkeeping; the device stream keeps its own
// history in HBM, see ppfg_stream_*)
inline SampleBlock carry_history(StreamState& state, const SampleBlock& block, std::size_t n_taps) {
    if (n_taps == 0)
        throw config_error("carry_history: n_taps must be >= 1");
    const std::size_t nc = block.n_channels;
    SampleBlock joined;
    joined.n_channels = nc;
    detail::reserve_huge(joined.samples, state.history.size() + block.samples.size());
    joined.samples.insert(joined.samples.end(), state.history.begin(), state.history.end());
    joined.samples.insert(joined.samples.end(), block.samples.begin(), block.samples.end());
    const std::size_t avail = joined.samples.size() / (nc ? nc : 1);
    const std::size_t keep = std::min(n_taps - 1, avail) * nc;
    state.history.assign(joined.samples.end() - static_cast<std::ptrdiff_t>(keep), joined.samples.end());
    return joined;
}

struct StreamOptions {
    unsigned workers = 1;
    bool zero_prime = false;
    const FilterCoefficients* coefficients = nullptr;
};

// pipeline.hpp:89-200 over the device-resident stream (ppfg_process_stream)
inline StreamState process_stream(const PpfConfig& config, std::istream& source, std::ostream& sink,
                                  const StreamOptions& options = {}) {
    config.validate();
    if (options.workers == 0)
        throw config_error("process_stream: workers must be >= 1");
    FilterCoefficients coeffs;
    if (options.coefficients) {
        if (options.coefficients->n_channels != config.n_channels ||
            options.coefficients->n_taps != config.n_taps)
            throw config_error("process_stream: supplied coefficients do not match the config");
        coeffs = *options.coefficients;
    } else {
        coeffs = generate_prototype(config.n_channels, config.n_taps, config.window);
    }
    Plan p(config.n_channels, config.n_taps, coeffs.values.data());
    // the callbacks run on library threads: an exception thrown by the
    // istream / ostream (exceptions() enabled) is caught there, kept, and
    // rethrown here once the library has returned
    struct Io {
        std::istream* is;
        std::ostream* os;
        std::exception_ptr read_exc, write_exc;
    } io{&source, &sink, nullptr, nullptr};
    auto rd = [](void* ctx, void* buf, std::uint64_t n) -> std::int64_t {
        auto& c = *static_cast<Io*>(ctx);
        try {
            c.is->read(static_cast<char*>(buf), static_cast<std::streamsize>(n));
            const std::streamsize got = c.is->gcount();
            if (got > 0) // a partial read is processed first (pipeline.hpp:138-143)
                return static_cast<std::int64_t>(got);
            return c.is->bad() ? -1 : 0;
        } catch (...) {
            if (c.is->gcount() > 0) { // keep the delivered bytes; fail on the next read
                c.read_exc = std::current_exception();
                return static_cast<std::int64_t>(c.is->gcount());
            }
            c.read_exc = std::current_exception();
            return -1;
        }
    };
    auto wr = [](void* ctx, const void* buf, std::uint64_t n) -> int {
        auto& c = *static_cast<Io*>(ctx);
        try {
            c.os->write(static_cast<const char*>(buf), static_cast<std::streamsize>(n));
            return *c.os ? 0 : 1;
        } catch (...) {
            c.write_exc = std::current_exception();
            return 1;
        }
    };
    ppfg_stream_state st{};
    const int rc = ppfg_process_stream(p.get(), config.block_spectra, options.zero_prime ? 1 : 0,
                                       config.fft_fallback ? 1 : 0, rd, &io, wr, &io, &st);
    if (rc == PPFG_IO_ERROR && io.write_exc)
        std::rethrow_exception(io.write_exc);
    if (rc == PPFG_DECODE_ERROR && io.read_exc)
        std::rethrow_exception(io.read_exc);
    detail::check(rc);
    sink.flush();
    if (!sink)
        throw io_error("process_stream: sink flush failed");
    StreamState out;
    out.spectra_processed = st.spectra_processed;
    out.bytes_in = st.bytes_in;
    out.bytes_out = st.bytes_out;
    out.dropped_samples = st.dropped_samples;
    return out;
}

} // namespace PPF_GPU_NS
