// Narrow-tile strided instances (W forced to 2 or 4 columns): used by
// launches with too few default tiles to fill the SMs (batch-1 signals, e.g.
// BASELINE config 1's 2^20 calls), where more, smaller tiles balance the
// work across 148 SMs and keep several CTAs resident per SM.  The permutation-
// free path's strided kinds only (DIF, DIT-conj); fp64 and fp32.
#include "../pass.cuh"
#include "../registry.h"

namespace pafft_b200 {

#define PAFFT_NENTRY(T, PREC, RADIX, F0, F1, F2, F3, KIND, WV)                                                  \
    if constexpr (TilePolicy<T, Fac<F0, F1, F2, F3>, MAP_STRIDED, WV>::NTB <= 1024 &&                           \
                  TilePolicy<T, Fac<F0, F1, F2, F3>, MAP_STRIDED, WV>::SMEM <= 232448)                          \
        reg.push_back({PREC, RADIX, F0 * F1 * F2 * F3, F0, F1, F2, F3, KIND, MAP_STRIDED,                       \
                       TilePolicy<T, Fac<F0, F1, F2, F3>, MAP_STRIDED, WV>::W,                                  \
                       TilePolicy<T, Fac<F0, F1, F2, F3>, MAP_STRIDED, WV>::NTB,                                \
                       TilePolicy<T, Fac<F0, F1, F2, F3>, MAP_STRIDED, WV>::SMEM,                               \
                       (const void*)&pass_kernel<T, RADIX, F0, F1, F2, F3, KIND, MAP_STRIDED, WV>, WV});
#define PAFFT_NADD(T, PREC, RADIX, F0, F1, F2, F3, WV)                \
    PAFFT_NENTRY(T, PREC, RADIX, F0, F1, F2, F3, KIND_DIF, WV)        \
    PAFFT_NENTRY(T, PREC, RADIX, F0, F1, F2, F3, KIND_DIT_CONJ, WV)
// strided stage groups of 2^20-point (radix 2/4) and 3^k / 5^k signals
#define PAFFT_NARROW_SHAPES(X, T, PREC, WV)                                                          \
    X(T, PREC, 2, 16, 16, 1, 1, WV) X(T, PREC, 2, 8, 8, 8, 1, WV) X(T, PREC, 2, 16, 8, 8, 1, WV)       \
    X(T, PREC, 4, 16, 16, 1, 1, WV) X(T, PREC, 4, 16, 16, 4, 1, WV)

void register_narrow_f64(Registry& reg) {
    PAFFT_NARROW_SHAPES(PAFFT_NADD, double, 0, 2)
    PAFFT_NARROW_SHAPES(PAFFT_NADD, double, 0, 4)
}
void register_narrow_f32(Registry& reg) {
    PAFFT_NARROW_SHAPES(PAFFT_NADD, float, 1, 4)
    PAFFT_NARROW_SHAPES(PAFFT_NADD, float, 1, 8)
}

}  // namespace pafft_b200
