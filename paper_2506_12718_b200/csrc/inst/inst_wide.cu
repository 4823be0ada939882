// Wide strided instances (fp64): 16 columns = 256-byte row segments instead of
// the default 8.  Taken by launches with many tiles (use_wide,
// pafft_b200.cu), where the longer HBM row segments pay (config 4's 256^3
// axis-1/2 passes: +4% conv/s); batch-1 launches keep 8 columns (config 1's
// 2^20 signal: 512 default tiles, -8% with 16 columns).
#include "../pass.cuh"
#include "../registry.h"

namespace pafft_b200 {

#define PAFFT_WENTRY(RADIX, F0, F1, F2, F3, KIND)                                                           \
    if constexpr (TilePolicy<double, Fac<F0, F1, F2, F3>, MAP_STRIDED, 16>::NTB <= 1024 &&                  \
                  TilePolicy<double, Fac<F0, F1, F2, F3>, MAP_STRIDED, 16>::SMEM <= 232448)                 \
        reg.push_back({0, RADIX, F0 * F1 * F2 * F3, F0, F1, F2, F3, KIND, MAP_STRIDED,                       \
                       TilePolicy<double, Fac<F0, F1, F2, F3>, MAP_STRIDED, 16>::W,                          \
                       TilePolicy<double, Fac<F0, F1, F2, F3>, MAP_STRIDED, 16>::NTB,                        \
                       TilePolicy<double, Fac<F0, F1, F2, F3>, MAP_STRIDED, 16>::SMEM,                       \
                       (const void*)&pass_kernel<double, RADIX, F0, F1, F2, F3, KIND, MAP_STRIDED, 16>, 1});
#define PAFFT_WADD(RADIX, F0, F1, F2, F3)                  \
    PAFFT_WENTRY(RADIX, F0, F1, F2, F3, KIND_DIF)          \
    PAFFT_WENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_CONJ)     \
    PAFFT_WENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_FWD)

// the 256-point (radix 2/4) and 243/125/64-point strided groups whose 16-column
// double-buffered tiles fit one SM
void register_wide_f64(Registry& reg) {
    PAFFT_WADD(2, 16, 16, 1, 1)
    PAFFT_WADD(4, 16, 16, 1, 1)
    PAFFT_WADD(2, 8, 8, 1, 1)
    PAFFT_WADD(4, 16, 4, 1, 1)
    PAFFT_WADD(8, 8, 8, 1, 1)
}

}  // namespace pafft_b200
