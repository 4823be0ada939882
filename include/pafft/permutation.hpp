// pafft/permutation.hpp -- drop-in for the reference's digit-reversal API
// (reference include/pafft/permutation.hpp:9-27).  The reordering runs on the
// device (tiled digit-reversal transposition); the pass counter is
// thread-local and counts whole-buffer reorderings exactly as the reference's
// (permutation.cpp:10): prepare_filter 1, convolve_standard 2, convolve_permfree 0.
#pragma once

#include <cstdint>

#include "core.hpp"

namespace pafft {

// Base-r digit reversal of j over `digits` positions; IndexOutOfRange when
// j >= r^digits.
inline std::uint64_t digit_reverse(std::uint64_t j, unsigned radix, unsigned digits) {
    std::uint64_t out = 0;
    detail::check(pafft_digit_reverse(j, radix, digits, &out));
    return out;
}

// Whole-tensor reordering: (i_1..i_d) <-> (rev(i_1)..rev(i_d)), one pass.
inline void permute_tensor(ComplexBuffer& x, const Plan& plan) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), 5, x.re.data(), x.im.data(), 1));
}

// Reordering of one standalone line of dimension `dim`.
inline void permute_1d(ComplexBuffer& x, const Plan& plan, std::size_t dim) {
    const std::size_t n = plan.shape().dim(dim);
    if (x.size() != n) throw ShapeMismatch(n, x.size());
    const Plan line(plan.radix(dim), TensorShape{n});
    detail::check(pafft_transform_split(line.handle(), 5, x.re.data(), x.im.data(), 1));
}

inline std::uint64_t permutation_pass_count() { return pafft_permutation_pass_count(); }
inline void reset_permutation_pass_count() { pafft_reset_permutation_pass_count(); }

}  // namespace pafft
