// stream_bench: end-to-end throughput of the drop-in process_stream (the
// reference's `ppf run` path, pipeline.hpp:89-200) over in-memory streams:
// source = istream over a synthetic byte string, sink = a counting streambuf.
// Usage: stream_bench [C=1024] [T=8] [MiB=2048] [block_spectra=4096]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <streambuf>
#include <string>
#include <vector>

#include "ppf_gpu/ppf.hpp"

namespace {
struct CountBuf : std::streambuf {
    unsigned long long n = 0;
    std::streamsize xsputn(const char*, std::streamsize k) override {
        n += static_cast<unsigned long long>(k);
        return k;
    }
    int_type overflow(int_type c) override {
        ++n;
        return c;
    }
};
struct MemBuf : std::streambuf {
    MemBuf(char* b, size_t n) { setg(b, b, b + n); }
};
} // namespace

int main(int argc, char** argv) {
    const std::size_t C = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1024;
    const std::size_t T = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 8;
    const std::size_t mib = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 2048;
    const std::size_t block = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 4096;
    const std::size_t S = (mib << 20) / (C * 8);
    std::vector<char> data(S * C * 8);
    if (ppfg_synth(C, 1, 0, S * C, data.data(), PPFG_MEM_HOST, 0, nullptr) != PPFG_OK) {
        std::fprintf(stderr, "synth failed\n");
        return 1;
    }
    ppf_gpu::PpfConfig cfg;
    cfg.n_channels = C;
    cfg.n_taps = T;
    cfg.block_spectra = block;
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
        MemBuf mb(data.data(), data.size());
        std::istream is(&mb);
        CountBuf cb;
        std::ostream os(&cb);
        const auto t0 = std::chrono::steady_clock::now();
        const auto st = ppf_gpu::process_stream(cfg, is, os);
        const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (st.bytes_out != cb.n) {
            std::fprintf(stderr, "byte count mismatch\n");
            return 1;
        }
        best = t < best ? t : best;
    }
    std::printf("{\"path\": \"process_stream (drop-in, EXACT)\", \"C\": %zu, \"T\": %zu, \"block_spectra\": %zu, "
                "\"bytes_in\": %zu, \"seconds\": %.4f, \"gb_per_s_in\": %.3f, \"x_realtime\": %.2f}\n",
                C, T, block, data.size(), best, data.size() / best / 1e9, data.size() / best / 6.5e9);
    return 0;
}
