// pafft/butterfly.hpp -- drop-in for the reference's stage-ladder API
// (reference include/pafft/butterfly.hpp:7-37): the three ladder flavours
// over a line or over every mode of a tensor.  On the device a tensor ladder
// is a sequence of per-axis stage-group passes with no transposes
// (DESIGN.md 3); the ladder semantics (stage order, twiddle placement,
// unnormalised) are the reference's.
#pragma once

#include "core.hpp"

namespace pafft {

enum class ButterflyVariant {
    forward,     // A: ascending stages, digit-reversed input -> DFT
    conjugate,   // A-bar: the conjugate ladder (inverse up to 1/n)
    transposed,  // A^T: descending stages, natural input -> digit-reversed DFT
};

// The radix-8 kernels' scaled eighth roots a = (1 - i)/sqrt(2), b = -i a.
struct Radix8Constants {
    static constexpr double inv_sqrt2 = 0.70710678118654752440;
    static constexpr double a_re = inv_sqrt2, a_im = -inv_sqrt2;
    static constexpr double b_re = -inv_sqrt2, b_im = -inv_sqrt2;
};

namespace detail {
// pafft_transform_split op codes of the three ladders
inline int ladder_op(ButterflyVariant v) {
    switch (v) {
        case ButterflyVariant::forward: return 2;
        case ButterflyVariant::transposed: return 4;
        default: return 6;
    }
}
inline void ladder_line(ComplexBuffer& x, const Plan& plan, std::size_t dim, ButterflyVariant v) {
    const std::size_t n = plan.shape().dim(dim);
    if (x.size() != n) throw ShapeMismatch(n, x.size());
    if (n < 2) return;
    const Plan line(plan.radix(dim), TensorShape{n});
    check(pafft_transform_split(line.handle(), ladder_op(v), x.re.data(), x.im.data(), 1));
}
}  // namespace detail

inline void butterfly_forward(ComplexBuffer& x, const Plan& plan, std::size_t dim) {
    detail::ladder_line(x, plan, dim, ButterflyVariant::forward);
}
inline void butterfly_conjugate(ComplexBuffer& x, const Plan& plan, std::size_t dim) {
    detail::ladder_line(x, plan, dim, ButterflyVariant::conjugate);
}
inline void butterfly_transposed(ComplexBuffer& x, const Plan& plan, std::size_t dim) {
    detail::ladder_line(x, plan, dim, ButterflyVariant::transposed);
}
// Kept from the previous drop-in (a line of dimension `dim`, any variant).
inline void butterfly_line(ComplexBuffer& x, const Plan& plan, std::size_t dim, ButterflyVariant variant) {
    detail::ladder_line(x, plan, dim, variant);
}

inline void butterfly_tensor(ComplexBuffer& x, const Plan& plan, ButterflyVariant variant) {
    if (x.size() != plan.total()) throw LengthMismatch(plan.total(), x.size());
    detail::check(pafft_transform_split(plan.handle(), detail::ladder_op(variant), x.re.data(), x.im.data(), 1));
}

}  // namespace pafft
