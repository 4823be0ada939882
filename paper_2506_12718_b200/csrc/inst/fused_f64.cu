// Fused permutation-free convolution instances (fused.cuh), fp64: one per
// (radix, strided split, contiguous split) the 1-D BASELINE plans use.
#include "../fused.cuh"
#include "../registry.h"

namespace pafft_b200 {

#define PAFFT_FUSED(RADIX, D0, D1, D2, D3, WD, C0, C1, C2, C3, WC)                                            \
    {                                                                                                          \
        using SH = FusedShape<double, RADIX, D0, D1, D2, D3, WD, C0, C1, C2, C3, WC>;                          \
        static_assert(SH::SMEM <= 232448, "fused tile shapes exceed shared memory");                         \
        reg.push_back({0, RADIX, D0 * D1 * D2 * D3, C0 * C1 * C2 * C3, WD, WC, SH::NT, SH::SMEM,             \
                       (const void*)&fused_conv_kernel<double, RADIX, D0, D1, D2, D3, WD, C0, C1, C2, C3, WC>}); \
    }

void register_fused_f64(FusedRegistry& reg) {
    PAFFT_FUSED(3, 9, 9, 9, 1, 8, 9, 9, 9, 3, 3)       // config 2: 3^13 = 729 x 2187
    PAFFT_FUSED(5, 25, 1, 1, 1, 128, 25, 25, 5, 1, 1)  // config 5: 5^7 = 25 x 3125
    PAFFT_FUSED(2, 16, 16, 1, 1, 16, 16, 16, 16, 1, 1)  // config 1: 2^20 = 256 x 4096
}

}  // namespace pafft_b200
