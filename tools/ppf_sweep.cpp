// ppf_sweep — the reference's `ppf bench --sweep` report (bench.hpp sweep /
// to_json / to_csv_row, cli.hpp:191-246) through the GPU drop-in, with the
// roofline columns: the taps sweep (C = 1024, T = 4..64) and the channels
// sweep (T = 8, C = 64..8192) of BASELINE.json, one CSV row and one JSON line
// per shape (the paper's Figure-2 table plus the HBM-roofline fraction).
//
//   tools/ppf_sweep [total_mib=512] [reps=3] [hbm_peak_gbs=0 (device theoretical)]
#include <cstdio>
#include <cstdlib>
#include <iostream>

#include "ppf_gpu/bench.hpp"

int main(int argc, char** argv) {
    const std::uint64_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 512;
    ppf_gpu::BenchOptions opt;
    opt.repetitions = argc > 2 ? static_cast<unsigned>(std::strtoul(argv[2], nullptr, 10)) : 3;
    opt.hbm_peak_gb_per_sec = argc > 3 ? std::strtod(argv[3], nullptr) : 0.0;
    std::vector<std::pair<std::size_t, std::size_t>> shapes;
    for (std::size_t T : {4, 8, 16, 32, 64})
        shapes.emplace_back(1024, T);
    for (std::size_t C : {64, 128, 256, 512, 2048, 4096, 8192})
        shapes.emplace_back(C, 8);
    ppf_gpu::PpfConfig base;
    base.n_channels = 1024;
    base.n_taps = 8;
    const auto entries = ppf_gpu::sweep(base, shapes, mib << 20, 1, opt);
    std::printf("%s,kernel\n", ppf_gpu::csv_header_roofline().c_str());
    for (const auto& e : entries) {
        if (e.report)
            std::printf("%s,%s\n", ppf_gpu::to_csv_row_roofline(*e.report).c_str(), e.report->kernel.c_str());
        else
            std::printf("%zu,%zu,error: %s\n", e.n_channels, e.n_taps, e.error.c_str());
    }
    for (const auto& e : entries)
        if (e.report)
            std::cerr << ppf_gpu::to_json(*e.report).dump() << "\n";
    return 0;
}
