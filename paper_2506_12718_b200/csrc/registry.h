// Kernel registry: every compiled pass-kernel instance, keyed by
// (precision, radix, R, kind).  The host plan (pafft_b200.cu) picks one per
// stage group; R = R1 * R2 * R3 is the in-tile codelet split.
#pragma once

#include <vector>

namespace pafft_b200 {

struct KernelEntry {
    int prec;   // 0 = f64, 1 = f32
    int radix;
    int R, F0, F1, F2, F3;  // codelet split R = F0 F1 F2 F3
    int kind;   // PassKind
    int map;    // PassMap
    int W, NT, smem;  // compile-time tile policy of this instance
    const void* fn;
    int wide = 0;     // 1: wide strided variant (more columns per tile) for launches with many tiles;
                      // 2: dense fp32 strided variant (even row lengths, tensor maps, no spare row slots)
};

using Registry = std::vector<KernelEntry>;

void register_r2_f64(Registry&);
void register_r3_f64(Registry&);
void register_r4_f64(Registry&);
void register_r5_f64(Registry&);
void register_r8_f64(Registry&);
void register_r2_f32(Registry&);
void register_r3_f32(Registry&);
void register_r4_f32(Registry&);
void register_r5_f32(Registry&);
void register_r8_f32(Registry&);
void register_wide_f64(Registry&);


}  // namespace pafft_b200

// Codelet splits per radix: each factor is a power of the radix so the
// digit reversal splits per step (pass.cuh).  R = F0 * F1 * F2 * F3.
#define PAFFT_SHAPES_R2(X)                                                                                    \
    X(2, 2, 1, 1, 1) X(2, 4, 1, 1, 1) X(2, 8, 1, 1, 1) X(2, 16, 1, 1, 1) X(2, 32, 1, 1, 1) X(2, 8, 8, 1, 1)     \
    X(2, 16, 8, 1, 1) X(2, 16, 16, 1, 1) X(2, 8, 8, 8, 1) X(2, 16, 8, 8, 1) X(2, 16, 16, 8, 1)                  \
    X(2, 16, 16, 16, 1)
#define PAFFT_SHAPES_R4(X) \
    X(4, 4, 1, 1, 1) X(4, 16, 1, 1, 1) X(4, 16, 4, 1, 1) X(4, 16, 16, 1, 1) X(4, 16, 16, 4, 1) X(4, 16, 16, 16, 1)
#define PAFFT_SHAPES_R8(X) X(8, 8, 1, 1, 1) X(8, 8, 8, 1, 1) X(8, 8, 8, 8, 1) X(8, 8, 8, 8, 8)
#define PAFFT_SHAPES_R3(X)                                                                                    \
    X(3, 3, 1, 1, 1) X(3, 9, 1, 1, 1) X(3, 27, 1, 1, 1) X(3, 9, 9, 1, 1) X(3, 9, 9, 3, 1) X(3, 9, 9, 9, 1)      \
    X(3, 9, 9, 9, 3) X(3, 9, 9, 9, 9)
#define PAFFT_SHAPES_R5(X) X(5, 5, 1, 1, 1) X(5, 25, 1, 1, 1) X(5, 5, 5, 5, 1) X(5, 5, 5, 5, 5) X(5, 25, 25, 5, 1)
