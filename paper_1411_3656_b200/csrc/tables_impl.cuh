// tables_impl.cuh — helpers that turn kernel configurations into table
// entries; included only by the tab_*.cu translation units.
#pragma once

#include "tables.h"

#include "dft.cuh"
#include "fft.cuh"
#include "fir.cuh"
#include "fused.cuh"
#include "fused_split.cuh"
#include "tiny.cuh"
#include "l2x.cuh"

namespace ppfg {

// The detection variant exists where every FFT thread's last-pass units see
// the same bins (FusedCfg::POWER_OK), so its accumulators stay per bin.
template <class Cfg>
constexpr bool has_power() {
    return Cfg::POWER_OK;
}

template <class Cfg>
FusedEntry fused_entry() {
    FusedEntry e{Cfg::L,    Cfg::T,  Cfg::EXACT, reinterpret_cast<KernelFn>(&fused_fir_fft_kernel<Cfg>),
                 Cfg::SMEM, Cfg::NT, Cfg::B * Cfg::G, 1, true};
    e.tw4 = Cfg::TW4;
    e.sig = __PRETTY_FUNCTION__;
    if constexpr (has_power<Cfg>()) {
        e.power_fn = reinterpret_cast<KernelFn>(&fused_fir_fft_kernel<Cfg, true>);
        e.power_rows = Cfg::POWER_ROWS;
    }
    return e;
}

// A configuration used for detection only (fir_fft_mean_power): its register
// split / FFT warpgroups are chosen for the accumulating last pass
template <class Cfg>
FusedEntry power_entry() {
    static_assert(has_power<Cfg>(), "detection variant");
    FusedEntry e = fused_entry<Cfg>();
    e.power_only = true;
    return e;
}

template <class Cfg>
FusedEntry split_entry(bool preferred) {
    FusedEntry e{Cfg::L,    Cfg::T,  Cfg::EXACT, reinterpret_cast<KernelFn>(&fused_split_kernel<Cfg>),
                 Cfg::SMEM, Cfg::NT, Cfg::B,     Cfg::Q,
                 preferred, Cfg::MAP_R, Cfg::RB, Cfg::MAP_RUN, Cfg::MAP_BOX_R};
    e.tw4 = Cfg::TW4;
    e.sig = __PRETTY_FUNCTION__;
    if constexpr (Cfg::POWER_OK) {
        e.power_fn = reinterpret_cast<KernelFn>(&fused_split_kernel<Cfg, true>);
        e.power_rows = Cfg::POWER_ROWS;
    }
    return e;
}

// Which (C, T) get a fused kernel. Register budget per SM ~ C * (3T fp32 |
// 6T fp64) for the FIR windows + taps, plus the FFT pass registers. Entries
// with (120, 80, 2, 3) run three FFT warpgroups (640 threads): measured faster
// where the FFT role is critical (C=1024/T=8, C=64, T=1 at C<=128), slower

} // namespace ppfg
