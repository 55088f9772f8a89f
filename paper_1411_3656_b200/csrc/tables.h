// tables.h — kernel dispatch tables of libppfg.so. The kernel instantiations
// live in separate translation units (tab_*.cu) so nvcc compiles them in
// parallel; ppfg.cu (host code) only sees these descriptors.
#pragma once

#include <cstddef>
#include <vector>

namespace ppfg {

using KernelFn = const void*;

struct FusedEntry {
    int L, T;
    bool exact;
    KernelFn fn;
    size_t smem;
    int nt;
    int rows_per_batch; // B * G
    int q;              // CTAs per cluster (1: single-SM kernel)
    bool preferred;     // cluster kernels: faster than FIR -> HBM -> FFT (measured)
    int map_r = 0;      // > 0: the kernel reads its input through a 3-D TMA tensor
    int map_rb = 0;     //      map of map_r runs of C/map_r channels, box {map_run,
    int map_run = 0;    //      map_box_r, map_rb} (fused_split.cuh)
    int map_box_r = 0;
    KernelFn power_fn = nullptr; // detection variant (POWER), single-SM entries
    int power_rows = 0;          // its partials per CTA (tile rows)
    bool tw4 = false;            // takes the pre-expanded float4 twiddle table
    const char* sig = nullptr;   // __PRETTY_FUNCTION__ of the entry maker: names the Cfg
    bool power_only = false;     // a detection-only configuration (power_fn; fn unused)
};

struct FftEntry {
    KernelFn fn;
    size_t smem;
    int nt;
    int rows_per_tile;
};

// K2n tile FFT (fft.cuh fft_tiles_kernel) for 6 <= L <= 13, or {} if none
FftEntry fft_tiles_entry(int L);

constexpr int kFftW = 5;
constexpr int kFftNT = 256;
constexpr int kFftMaxL = 13;

struct FirEntry {
    KernelFn fn;
    int tc, k; // taps per lane, lanes per channel (T = tc * k)
};

// K1 variants: one lane per channel up to T = 16; larger T split over K
// lanes of up to 16 taps (T = TC * K), chained with a lag (fir.cuh).
struct FirTmaEntry {
    KernelFn fn = nullptr;
    int k = 0, rb = 0;
    size_t smem = 0;
};

// K1b shapes (register-blocked, CTA-wide TMA ring; fir.cuh): U = 16 outputs
// per thread, 4 warps per CTA
struct FirBlkEntry {
    KernelFn fn = nullptr;
    int rb = 0, nt = 0;
    size_t smem = 0;
};

// The fused table in dispatch order (first match wins): the parts below,
// concatenated by fused_table() in ppfg.cu.
std::vector<FusedEntry> fused_part_main();   // tab_fused_main.cu
std::vector<FusedEntry> fused_part_small();  // tab_fused_small.cu
std::vector<FusedEntry> fused_part_fft();    // tab_fused_fft.cu
std::vector<FusedEntry> fused_part_split();  // tab_split.cu

const FftEntry* fft_table(int L);   // K2, tab_fft.cu
FirTmaEntry fir_tma_table(int T);   // K1t, tab_fir.cu
FirTmaEntry fir_fast_table(int T);  // K1f, tab_fir.cu
FirBlkEntry fir_blk_table(int T, bool exact); // K1b, tab_fir_blk.cu
FirEntry fir_table(int T);          // K1, tab_fir.cu
// K7 fused FIR + FFT through an L2-resident exchange ring (l2x.cuh)
struct L2xEntry {
    int L, T;
    bool exact;
    KernelFn fn;
    size_t smem;
    int nt;
    int rb;                    // TMA box rows (input chunk)
    size_t ring_bytes;         // the exchange ring in global memory
    int nsr;                   // ring slots (counters: 2 * nsr)
    bool preferred;            // taken by default (measured faster than the alternatives)
    const char* sig = nullptr; // __PRETTY_FUNCTION__ of the entry maker
};
std::vector<L2xEntry> l2x_table(); // tab_l2x.cu

// K6 fused FIR+FFT for C = 2^L, L = 0..5 (tiny.cuh), tab_tiny.cu; nullptr
// where no instantiation covers (L, T, exact)
KernelFn tiny_table(int L, int T, bool exact);
KernelFn fir_c1_table(int T); // K6 at C = 1 (fir_c1_kernel), tab_tiny.cu

} // namespace ppfg
