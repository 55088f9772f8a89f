// Drop-in process_stream with throwing streams: the callbacks
// run on library threads; an exception thrown by the istream / ostream must
// reach the caller (not std::terminate), and bytes delivered before a read
// failure must be processed first (pipeline.hpp:138-143). Exit 0 = pass.
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <streambuf>
#include <string>
#include <vector>

#include "ppf_gpu/ppf.hpp"

namespace {
// delivers `good` bytes (a whole number of the reader's requests), then fails
// the next read with an exception
struct FailingBuf : std::streambuf {
    std::string data;
    size_t pos = 0, good;
    explicit FailingBuf(std::string d, size_t g) : data(std::move(d)), good(g) {}
    std::streamsize xsgetn(char* s, std::streamsize n) override {
        if (pos >= good)
            throw std::runtime_error("source failed");
        const std::streamsize k = std::min<std::streamsize>(n, static_cast<std::streamsize>(good - pos));
        std::copy(data.data() + pos, data.data() + pos + k, s);
        pos += static_cast<size_t>(k);
        return k;
    }
    int_type underflow() override { return traits_type::eof(); }
};
struct FailingSink : std::streambuf {
    size_t n = 0, limit;
    explicit FailingSink(size_t l) : limit(l) {}
    std::streamsize xsputn(const char*, std::streamsize k) override {
        if (n + static_cast<size_t>(k) > limit)
            throw std::runtime_error("sink failed");
        n += static_cast<size_t>(k);
        return k;
    }
};
} // namespace

int main() {
    const std::size_t C = 64, T = 8, S = 4000;
    std::string src(S * C * 8, '\0');
    if (ppfg_synth(C, 1, 0, S * C, src.data(), PPFG_MEM_HOST, 0, nullptr) != PPFG_OK)
        return 2;
    ppf_gpu::PpfConfig cfg;
    cfg.n_channels = C;
    cfg.n_taps = T;
    cfg.block_spectra = 256;
    int failures = 0;
    { // 1. a throwing source (exceptions enabled on the istream): the exception reaches the caller
        FailingBuf fb(src, 4 * 256 * C * 8);
        std::istream is(&fb);
        is.exceptions(std::ios::badbit);
        std::ostringstream os;
        try {
            ppf_gpu::process_stream(cfg, is, os);
            std::printf("FAIL: no exception from a throwing source\n");
            ++failures;
        } catch (const std::exception& e) {
            // the reference would have processed the bytes before the failure
            if (os.str().size() != (4 * 256 - T + 1) * C * 8) {
                std::printf("FAIL: output before the source failure missing (%zu bytes)\n", os.str().size());
                ++failures;
            } else {
                std::printf("ok: source exception propagated (%s), %zu bytes written before it\n", e.what(),
                            os.str().size());
            }
        }
    }
    { // 2. a source that goes bad without exceptions: decode_error at the byte offset
        FailingBuf fb(src, 4 * 256 * C * 8);
        std::istream is(&fb);
        std::ostringstream os;
        try {
            ppf_gpu::process_stream(cfg, is, os);
            std::printf("FAIL: no decode_error from a failing source\n");
            ++failures;
        } catch (const ppf_gpu::decode_error& e) {
            if (e.byte_offset != 4 * 256 * C * 8) {
                std::printf("FAIL: decode_error offset %llu\n", static_cast<unsigned long long>(e.byte_offset));
                ++failures;
            } else {
                std::printf("ok: decode_error at byte %llu\n", static_cast<unsigned long long>(e.byte_offset));
            }
        }
    }
    { // 3. a throwing sink: the exception reaches the caller
        std::istringstream is(src);
        FailingSink sb(300 * C * 8);
        std::ostream os(&sb);
        os.exceptions(std::ios::badbit);
        try {
            ppf_gpu::process_stream(cfg, is, os);
            std::printf("FAIL: no exception from a throwing sink\n");
            ++failures;
        } catch (const std::exception& e) {
            std::printf("ok: sink exception propagated (%s)\n", e.what());
        }
    }
    return failures == 0 ? 0 : 1;
}
