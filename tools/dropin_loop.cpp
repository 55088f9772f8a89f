// dropin_loop: the reference's own per-block compute pass (bench.hpp:129-150:
// carry_history -> ppf_fir_optimized -> channelize_block on std::vectors)
// compiled against the GPU drop-in (ppf_gpu/ppf.hpp) — what a reference caller
// that loops per block gets without changing a line. Reports input GB/s of the
// whole loop, the time split (carry_history / FIR call / channelize call), the
// first (cold: plan creation) call vs the steady state, and the fixed per-call
// cost (the same calls on an 8-spectrum block) as a fraction of a full call.
//
//   tools/dropin_loop [C=1024] [T=8] [MiB=1024] [block_spectra=4096]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ppf_gpu/ppf.hpp"

namespace {
double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
} // namespace

int main(int argc, char** argv) {
    const std::size_t C = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1024;
    const std::size_t T = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 8;
    const std::size_t mib = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1024;
    const std::size_t bs = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 4096;
    const std::size_t S = (mib << 20) / (C * 8);
    std::vector<ppf_gpu::ComplexSample> samples(S * C);
    if (ppfg_synth(C, 1, 0, S * C, samples.data(), PPFG_MEM_HOST, 0, nullptr) != PPFG_OK)
        return 1;
    const auto coeffs = ppf_gpu::generate_prototype(C, T, ppf_gpu::WindowSpec{});
    const unsigned workers = 1;

    // cold: the first calls of the process (plan creation, staging allocation)
    double cold_fir = 0, cold_chan = 0;
    {
        ppf_gpu::SampleBlock b;
        b.n_channels = C;
        b.samples.assign(samples.begin(), samples.begin() + static_cast<std::ptrdiff_t>(bs * C));
        double t0 = now();
        const auto f = ppf_gpu::ppf_fir_optimized(b, coeffs, workers);
        cold_fir = now() - t0;
        t0 = now();
        const auto o = ppf_gpu::channelize_block(f, true, workers);
        cold_chan = now() - t0;
    }
    auto pass = [&](std::size_t block_spectra, double* t_carry, double* t_fir, double* t_chan) {
        ppf_gpu::StreamState state;
        ppf_gpu::SampleBlock block;
        block.n_channels = C;
        std::uint64_t emitted = 0;
        for (std::size_t s = 0; s < S; s += block_spectra) {
            const std::size_t n = std::min(block_spectra, S - s);
            double t0 = now();
            block.samples.assign(samples.begin() + static_cast<std::ptrdiff_t>(s * C),
                                 samples.begin() + static_cast<std::ptrdiff_t>((s + n) * C));
            const ppf_gpu::SampleBlock joined = ppf_gpu::carry_history(state, block, T);
            double t1 = now();
            *t_carry += t1 - t0;
            if (joined.n_spectra() < T)
                continue;
            const auto filtered = ppf_gpu::ppf_fir_optimized(joined, coeffs, workers);
            double t2 = now();
            *t_fir += t2 - t1;
            const auto chan = ppf_gpu::channelize_block(filtered, true, workers);
            *t_chan += now() - t2;
            emitted += chan.n_spectra;
        }
        return emitted;
    };
    double best = 1e30, bc = 0, bf = 0, bh = 0;
    for (int rep = 0; rep < 3; ++rep) {
        double tc = 0, tf = 0, th = 0;
        const double t0 = now();
        pass(bs, &tc, &tf, &th);
        const double t = now() - t0;
        if (t < best) {
            best = t;
            bc = tc;
            bf = tf;
            bh = th;
        }
    }
    const std::size_t n_blocks = (S + bs - 1) / bs;
    // fixed per-call cost: the same two calls on an 8-spectrum block
    double small = 1e30;
    {
        ppf_gpu::SampleBlock b;
        b.n_channels = C;
        b.samples.assign(samples.begin(), samples.begin() + static_cast<std::ptrdiff_t>((T + 7) * C));
        for (int rep = 0; rep < 20; ++rep) {
            const double t0 = now();
            const auto f = ppf_gpu::ppf_fir_optimized(b, coeffs, workers);
            const auto o = ppf_gpu::channelize_block(f, true, workers);
            small = std::min(small, now() - t0);
        }
    }
    const double per_block = (bf + bh) / n_blocks;
    std::printf("{\"path\": \"reference per-block loop (bench.hpp:129-150) through the drop-in\", "
                "\"C\": %zu, \"T\": %zu, \"block_spectra\": %zu, \"bytes_in\": %zu, \"seconds\": %.4f, "
                "\"gb_per_s_in\": %.3f, \"x_realtime\": %.3f, \"split_s\": {\"carry_history\": %.4f, "
                "\"ppf_fir_optimized\": %.4f, \"channelize_block\": %.4f}, "
                "\"cold_first_calls_s\": {\"ppf_fir_optimized\": %.4f, \"channelize_block\": %.4f}, "
                "\"fixed_per_call_pair_s\": %.6f, \"gpu_calls_per_block_s\": %.6f, "
                "\"per_call_overhead_frac\": %.4f}\n",
                C, T, bs, S * C * 8, best, S * C * 8 / best / 1e9, S * C * 8 / best / 6.5e9, bc, bf, bh,
                cold_fir, cold_chan, small, per_block, small / per_block);
    return 0;
}
