// Explicit pass-kernel instances: radix 5, double.
#include "../pass.cuh"
#include "../registry.h"

namespace pafft_b200 {

#define PAFFT_ADD(RADIX, R1, R2, R3)                                                                       \
    reg.push_back({0, RADIX, R1 * R2 * R3, R1, R2, R3, KIND_DIF,                                           \
                   (const void*)&pass_kernel<double, RADIX, R1, R2, R3, KIND_DIF>});                           \
    reg.push_back({0, RADIX, R1 * R2 * R3, R1, R2, R3, KIND_DIT_CONJ,                                      \
                   (const void*)&pass_kernel<double, RADIX, R1, R2, R3, KIND_DIT_CONJ>});                      \
    reg.push_back({0, RADIX, R1 * R2 * R3, R1, R2, R3, KIND_DIT_FWD,                                       \
                   (const void*)&pass_kernel<double, RADIX, R1, R2, R3, KIND_DIT_FWD>});                       \
    reg.push_back({0, RADIX, R1 * R2 * R3, R1, R2, R3, KIND_CONV,                                          \
                   (const void*)&pass_kernel<double, RADIX, R1, R2, R3, KIND_CONV>});

void register_r5_f64(Registry& reg) { PAFFT_SHAPES_R5(PAFFT_ADD) }

}  // namespace pafft_b200
