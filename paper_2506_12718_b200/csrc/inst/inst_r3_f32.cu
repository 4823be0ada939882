// Explicit pass-kernel instances: radix 3, float.
#include "../pass.cuh"
#include "../registry.h"

namespace pafft_b200 {

#define PAFFT_ENTRY(RADIX, R1, R2, R3, KIND, MAP)                                                       \
    reg.push_back({1, RADIX, R1 * R2 * R3, R1, R2, R3, KIND, MAP, TilePolicy<float, R1, R2, R3, MAP>::W,          \
                   TilePolicy<float, R1, R2, R3, MAP>::NT, TilePolicy<float, R1, R2, R3, MAP>::SMEM,                  \
                   (const void*)&pass_kernel<float, RADIX, R1, R2, R3, KIND, MAP>});
#define PAFFT_ADD(RADIX, R1, R2, R3)                                     \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_DIF, MAP_STRIDED)                \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_DIF, MAP_CONTIG)                 \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_DIT_CONJ, MAP_STRIDED)           \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_DIT_CONJ, MAP_CONTIG)            \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_DIT_FWD, MAP_STRIDED)            \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_DIT_FWD, MAP_CONTIG)             \
    PAFFT_ENTRY(RADIX, R1, R2, R3, KIND_CONV, MAP_CONTIG)

void register_r3_f32(Registry& reg) { PAFFT_SHAPES_R3(PAFFT_ADD) }

}  // namespace pafft_b200
