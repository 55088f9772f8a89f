// tab_l2x.cu — K7 fused FIR + FFT through an L2-resident exchange ring
// (l2x.cuh): long filters at C = 1024 and the C = 8192 transform.
#include "tables_impl.cuh"

namespace ppfg {

namespace {
template <class Cfg>
L2xEntry l2x_entry(bool preferred) {
    L2xEntry e{Cfg::L, Cfg::T, Cfg::EXACT, reinterpret_cast<KernelFn>(&fused_l2x_kernel<Cfg>),
               Cfg::SMEM, Cfg::NT, Cfg::RB, sizeof(float2) * Cfg::RING_SLOT_FLOATS2 * Cfg::NSR,
               Cfg::NSR, preferred};
    e.sig = __PRETTY_FUNCTION__;
    return e;
}
} // namespace

std::vector<L2xEntry> l2x_table() {
    return {
        // 8 FIR warps x 8 outputs per step (64-row TMA chunks, 4 in the ring),
        // 256-spectrum work items; 8 FFT warps in two groups, each with two
        // tile slots filled by TMA bulk copies of ring rows. Ring slots: the FIR role's round (one item
        // per CTA) fills grid / (C/32) = 4.6 chunks and the FFT role trails it
        // by a round, so 16 slots (32 MB) keep both roles busy
        l2x_entry<L2xCfg<10, 32, false, 8, 8, 4, 4, 16>>(false),
        l2x_entry<L2xCfg<10, 64, false, 8, 8, 4, 4, 16>>(false),
        l2x_entry<L2xCfg<10, 16, false, 8, 8, 4, 4, 16>>(false),
        l2x_entry<L2xCfg<10, 32, true, 8, 8, 4, 4, 16>>(false),
        // C = 8192: 64-spectrum items (4 MB ring slots), 4 slots, 4-chunk input ring
        // (one FFT group with one tile slot: two 8192-point tiles do not fit
        // next to the twiddles)
        l2x_entry<L2xCfg<13, 8, false, 8, 8, 1, 4, 4, 8, 5, 160, 96, 1, 1>>(false),
        l2x_entry<L2xCfg<13, 8, true, 8, 8, 1, 4, 4, 8, 5, 160, 96, 1, 1>>(false),
    };
}

} // namespace ppfg
