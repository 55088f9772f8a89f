// tab_fused_small.cu — K3 fused shapes for small C at T = 4, 16, 32.
#include "tables_impl.cuh"

namespace ppfg {

std::vector<FusedEntry> fused_part_small() {
    return {
        // small C at T = 4 and 16 (register budget: 3T·R FP32, 6T·R FP64 per FIR thread)
        fused_entry<FusedCfg<8, 16, 1, false, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<7, 16, 0, false, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<6, 16, 1, false, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<8, 16, 0, true, 160, 96, 4, 2, 2, false, 0, true, false, true>>(),
        fused_entry<FusedCfg<7, 16, 0, true, 160, 96, 4, 2, 2, false, 0, true, false, true>>(),
        fused_entry<FusedCfg<6, 16, 0, true, 160, 96, 4, 2, 2, false, 0, true, false, true>>(),
        fused_entry<FusedCfg<9, 4, 2, false>>(),
        fused_entry<FusedCfg<8, 4, 0, false, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<7, 4, 2, false>>(),
        fused_entry<FusedCfg<6, 4, 1, false>>(),
        fused_entry<FusedCfg<9, 4, 2, true, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<8, 4, 1, true, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<7, 4, 2, true, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<6, 4, 1, true, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<8, 32, 0, false, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<7, 32, 0, false, 160, 96, 4, 2, 2, false, 0, true>>(),
        fused_entry<FusedCfg<6, 32, 0, false, 160, 96, 4, 2, 2, false, 0, true>>(),
    };
}

} // namespace ppfg
