// Explicit pass-kernel instances: radix 4, float.
#include "../pass.cuh"
#include "../registry.h"

namespace pafft_b200 {

// instances whose tile policy cannot launch (> 1024 threads or > 227 KB of
// shared memory) are not registered; the plan then splits the axis further
#define PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND, MAP)                                                  \
    if constexpr (TilePolicy<float, Fac<F0, F1, F2, F3>, MAP>::NTB <= 1024 &&                                \
                  TilePolicy<float, Fac<F0, F1, F2, F3>, MAP>::SMEM <= 232448)                              \
        reg.push_back({1, RADIX, F0 * F1 * F2 * F3, F0, F1, F2, F3, KIND, MAP,                            \
                       TilePolicy<float, Fac<F0, F1, F2, F3>, MAP>::W, TilePolicy<float, Fac<F0, F1, F2, F3>, MAP>::NTB, \
                       TilePolicy<float, Fac<F0, F1, F2, F3>, MAP>::SMEM,                                          \
                       (const void*)&pass_kernel<float, RADIX, F0, F1, F2, F3, KIND, MAP>});
// dense strided instances (WOVR = -1) for even row lengths: registry variant 2
#define PAFFT_DENTRY(RADIX, F0, F1, F2, F3, KIND)                                                            \
    if constexpr (TilePolicy<float, Fac<F0, F1, F2, F3>, MAP_STRIDED, -1>::NTB <= 1024 &&                     \
                  TilePolicy<float, Fac<F0, F1, F2, F3>, MAP_STRIDED, -1>::SMEM <= 232448)                    \
        reg.push_back({1, RADIX, F0 * F1 * F2 * F3, F0, F1, F2, F3, KIND, MAP_STRIDED,                        \
                       TilePolicy<float, Fac<F0, F1, F2, F3>, MAP_STRIDED, -1>::W,                            \
                       TilePolicy<float, Fac<F0, F1, F2, F3>, MAP_STRIDED, -1>::NTB,                          \
                       TilePolicy<float, Fac<F0, F1, F2, F3>, MAP_STRIDED, -1>::SMEM,                         \
                       (const void*)&pass_kernel<float, RADIX, F0, F1, F2, F3, KIND, MAP_STRIDED, -1>, 2});
#define PAFFT_ADD(RADIX, F0, F1, F2, F3)                                     \
    PAFFT_DENTRY(RADIX, F0, F1, F2, F3, KIND_DIF)                            \
    PAFFT_DENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_CONJ)                       \
    PAFFT_DENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_FWD)                        \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_DIF, MAP_STRIDED)                \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_DIF, MAP_CONTIG)                 \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_CONJ, MAP_STRIDED)           \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_CONJ, MAP_CONTIG)            \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_FWD, MAP_STRIDED)            \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_DIT_FWD, MAP_CONTIG)             \
    PAFFT_ENTRY(RADIX, F0, F1, F2, F3, KIND_CONV, MAP_CONTIG)

void register_r4_f32(Registry& reg) { PAFFT_SHAPES_R4(PAFFT_ADD) }

}  // namespace pafft_b200
